"""Short driver for ncu: build one level and run a few fused evaluations.

    python tools/prof_eval.py [--n 256] [--ratio 4] [--evals 5] [--dtype f32] [--exact]
"""

import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_06765_b200 as ngf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--ratio", type=int, default=4)
    ap.add_argument("--evals", type=int, default=5)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--exact", action="store_true")
    a = ap.parse_args()
    dt = np.float32 if a.dtype == "f32" else np.float64
    R, T, _ = ngf.ct_pair(a.n, dtype=dt)
    gd = ngf.deformation_grid_for(R.grid, a.ratio)
    y = ngf.smooth_random_field(gd, seed=2, amplitude_mm=2.0).field.astype(dt)
    plan = ngf.build_gather_plan(gd, R.grid)
    obj = ngf.LevelObjective.from_device(torch.from_numpy(T.values).cuda(),
                                         torch.from_numpy(R.values).cuda(), plan, ngf.NgfParams(),
                                         1.0, exact=a.exact)
    x = torch.from_numpy(y.ravel().copy()).cuda()
    g = torch.empty_like(x)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(a.evals):
        sc = obj.eval_device(x, g)
    torch.cuda.synchronize()
    dt_ms = (time.perf_counter() - t0) * 1000 / a.evals
    print(f"n={a.n} ratio={a.ratio} {a.dtype} exact={a.exact}: {dt_ms:.3f} ms/eval, J={sc[0].item():.6g}")


if __name__ == "__main__":
    main()
