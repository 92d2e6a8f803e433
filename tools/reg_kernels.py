"""Per-kernel device time of one full registration (torch.profiler / CUPTI) and the
wall time, to split a registration into kernel time and host / latency gaps.

    python tools/reg_kernels.py [--n 256] [--levels 4]
"""

import argparse
import os
import sys
import time
from collections import defaultdict

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_06765_b200 as ngf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--levels", type=int, default=4)
a = ap.parse_args()
R, T, _ = ngf.ct_pair(a.n, dtype=np.float32)
cfg = ngf.MultilevelConfig(num_levels=a.levels, grid_ratio=4, precision="f32")
ngf.register(R, T, cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
ngf.register(R, T, cfg)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    ngf.register(R, T, cfg)
    torch.cuda.synchronize()
tot, cnt = defaultdict(float), defaultdict(int)
for e in prof.events():
    if e.device_type != torch.autograd.DeviceType.CUDA:
        continue
    k = e.name.split("(")[0][:60]
    tot[k] += e.device_time
    cnt[k] += 1
busy = sum(tot.values())
print(f"register {a.n}^3: wall {wall * 1e3:.1f} ms, kernels busy {busy / 1e3:.1f} ms")
for k in sorted(tot, key=lambda k: -tot[k])[:14]:
    print(f"  {k:60s} x{cnt[k]:<5d} {tot[k] / 1e3:8.2f} ms  ({tot[k] / cnt[k]:.1f} us each)")
