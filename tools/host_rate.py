"""Host issue rate of LevelObjective.eval_device (no profiler): wall time per call for
back-to-back calls vs the device time per evaluation.

    python tools/host_rate.py [--n 32]
"""

import argparse
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_06765_b200 as ngf  # noqa: E402
from paper_1812_06765_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32)
a = ap.parse_args()
R, T, _ = ngf.ct_pair(a.n, dtype=np.float32)
gd = ngf.deformation_grid_for(R.grid, 4)
y = ngf.smooth_random_field(gd, seed=2, amplitude_mm=2.0).field.astype(np.float32)
obj = ngf.LevelObjective.from_device(torch.from_numpy(T.values).cuda(), torch.from_numpy(R.values).cuda(),
                                     ngf.build_gather_plan(gd, R.grid), ngf.NgfParams(), 1.0)
x = torch.from_numpy(y.ravel().copy()).cuda()
g = torch.empty_like(x)
sc = torch.zeros(3, dtype=torch.float64, device="cuda")
lv = obj.level
h, s = lv.handle, torch.cuda.current_stream().cuda_stream
xp, gp, sp = x.data_ptr(), g.data_ptr(), sc.data_ptr()
for _ in range(20):
    obj.eval_device(x, g, sc)
torch.cuda.synchronize()
n = 500
t0 = time.perf_counter()
for _ in range(n):
    obj.eval_device(x, g, sc)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"{a.n}^3 eval_device: issue {(t1 - t0) / n * 1e6:.1f} us/call, total {(t2 - t0) / n * 1e6:.1f} us/eval")
lib = _lib.lib()
t0 = time.perf_counter()
for _ in range(n):
    lib.ngf_level_eval(h, xp, gp, sp, 0, s)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"{a.n}^3 raw ctypes ngf_level_eval: issue {(t1 - t0) / n * 1e6:.1f} us/call, total {(t2 - t0) / n * 1e6:.1f} us/eval")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n):
    lib.ngf_level_eval(h, xp, gp, sp, 0, s)
e1.record()
torch.cuda.synchronize()
print(f"device time per eval {e0.elapsed_time(e1) / n * 1e3:.1f} us")
