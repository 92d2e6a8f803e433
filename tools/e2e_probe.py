"""Break down the host-facing LevelObjective call (numpy in, numpy out) at 256^3 into its
pieces, timed on the host with the device synchronised.

    python tools/e2e_probe.py
"""

import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_06765_b200 as ngf  # noqa: E402


def t(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


R, T, _ = ngf.ct_pair(256, dtype=np.float32)
gd = ngf.deformation_grid_for(R.grid, 4)
y = ngf.smooth_random_field(gd, seed=2, amplitude_mm=2.0).field.astype(np.float32).ravel()
obj = ngf.LevelObjective.from_device(torch.from_numpy(T.values).cuda(), torch.from_numpy(R.values).cuda(),
                                     ngf.build_gather_plan(gd, R.grid), ngf.NgfParams(), 1.0)
obj(y)
x_dev, g_dev, sc_dev, sc_pin, x_pin = obj._stage
g_pin = torch.empty(y.size, dtype=torch.float32, pin_memory=True)
print(f"full __call__          {t(lambda: obj(y)):.3f} ms")
print(f"memcpy x -> pinned     {t(lambda: x_pin.numpy().__setitem__(slice(None), y)):.3f} ms")
print(f"H2D 3 MB               {t(lambda: x_dev.copy_(x_pin, non_blocking=True)):.3f} ms")
print(f"eval (device)          {t(lambda: obj.eval_device(x_dev, g_dev, sc_dev)):.3f} ms")
print(f"D2H 3 MB               {t(lambda: g_pin.copy_(g_dev, non_blocking=True)):.3f} ms")
print(f"pinned -> new array    {t(lambda: g_pin.numpy().copy()):.3f} ms")
print(f"scalars D2H + sync     {t(lambda: (sc_pin.copy_(sc_dev, non_blocking=True), torch.cuda.current_stream().synchronize())):.3f} ms")
xs = torch.from_numpy(y)
print(f"pageable H2D 3 MB      {t(lambda: x_dev.copy_(xs, non_blocking=False)):.3f} ms")
print(f"pinned alloc+D2H 3 MB  {t(lambda: torch.empty(y.size, dtype=torch.float32, pin_memory=True).copy_(g_dev, non_blocking=True)):.3f} ms")
