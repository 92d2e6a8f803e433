"""Time a full registration and break it down (pyramid, per-level setup / optimise)."""

import argparse
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_06765_b200 as ngf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--levels", type=int, default=4)
    ap.add_argument("--profile", action="store_true")
    a = ap.parse_args()
    R, T, _ = ngf.ct_pair(a.n, dtype=np.float32)
    cfg = ngf.MultilevelConfig(num_levels=a.levels, precision="f32")
    for it in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if a.profile and it == 2:
            pr = cProfile.Profile()
            pr.enable()
        y, rep = ngf.register(R, T, cfg)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if a.profile and it == 2:
            pr.disable()
            pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
        print(f"run {it}: {dt:.4f} s total (report {rep.seconds_total:.4f}); pyramid {rep.seconds_pyramid:.4f}")
        for lv in rep.levels:
            print(f"  level {lv.level_index} img {lv.image_dims[0]} def {lv.def_dims[0]}: setup "
                  f"{lv.seconds_setup:.4f} s, optimise {lv.seconds_optimize:.4f} s, {lv.iterations} it, "
                  f"{lv.evaluations} evals, {lv.stop_reason}")


if __name__ == "__main__":
    main()
