"""Host-side profile (cProfile) of a full registration: where the Python / ctypes /
torch time goes between kernels.

    python tools/prof_host.py [--n 128] [--levels 3]
"""

import argparse
import cProfile
import os
import pstats
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_06765_b200 as ngf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--levels", type=int, default=3)
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    R, T, _ = ngf.ct_pair(a.n, dtype=np.float32)
    cfg = ngf.MultilevelConfig(num_levels=a.levels, grid_ratio=4, precision="f32")
    ngf.register(R, T, cfg)
    t0 = time.perf_counter()
    y, rep = ngf.register(R, T, cfg)
    print(f"register {a.n}^3: {time.perf_counter() - t0:.4f} s, evals",
          [lv.evaluations for lv in rep.levels])
    pr = cProfile.Profile()
    pr.enable()
    ngf.register(R, T, cfg)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(a.top)


if __name__ == "__main__":
    main()
