"""Live per-kernel durations of one LevelObjective evaluation (torch.profiler / CUPTI,
no replay, warm caches), plus the wall span per evaluation.

    python tools/kernel_times.py [--n 256] [--ratio 4] [--evals 20] [--dtype f32]
"""

import argparse
import os
import sys
from collections import defaultdict

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_06765_b200 as ngf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--ratio", type=int, default=4)
    ap.add_argument("--evals", type=int, default=20)
    ap.add_argument("--dtype", default="f32")
    a = ap.parse_args()
    dt = np.float32 if a.dtype == "f32" else np.float64
    R, T, _ = ngf.ct_pair(a.n, dtype=dt)
    gd = ngf.deformation_grid_for(R.grid, a.ratio)
    y = ngf.smooth_random_field(gd, seed=2, amplitude_mm=2.0).field.astype(dt)
    plan = ngf.build_gather_plan(gd, R.grid)
    obj = ngf.LevelObjective.from_device(torch.from_numpy(T.values).cuda(),
                                         torch.from_numpy(R.values).cuda(), plan, ngf.NgfParams(), 1.0)
    x = torch.from_numpy(y.ravel().copy()).cuda()
    g = torch.empty_like(x)
    for _ in range(5):
        obj.eval_device(x, g)
    torch.cuda.synchronize()
    acts = [torch.profiler.ProfilerActivity.CUDA]
    with torch.profiler.profile(activities=acts) as prof:
        for _ in range(a.evals):
            obj.eval_device(x, g)
        torch.cuda.synchronize()
    tot = defaultdict(float)
    cnt = defaultdict(int)
    first = last = None
    for e in prof.events():
        if e.device_type != torch.autograd.DeviceType.CUDA:
            continue
        name = e.name.split("(")[0][:70]
        tot[name] += e.device_time
        cnt[name] += 1
        t0, t1 = e.time_range.start, e.time_range.end
        first = t0 if first is None else min(first, t0)
        last = t1 if last is None else max(last, t1)
    span = (last - first) / a.evals
    busy = sum(tot.values()) / a.evals
    print(f"n={a.n} ratio={a.ratio} {a.dtype}: span {span:.1f} us/eval, kernels busy {busy:.1f} us/eval")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"  {k:70s} x{cnt[k] // a.evals:<3d} {tot[k] / a.evals:9.1f} us/eval")


if __name__ == "__main__":
    main()
