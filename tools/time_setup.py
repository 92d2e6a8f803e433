"""Host cost of building one device level (plans, fused chunk planning, buffers, reference
terms) per image size.

    python tools/time_setup.py
"""

import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_06765_b200 as ngf  # noqa: E402

for n in (32, 64, 128, 256, 512):
    g = ngf.Grid3((n, n, n), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    gd = ngf.deformation_grid_for(g, 4)
    T = torch.zeros((n, n, n), dtype=torch.float32, device="cuda")
    plan = ngf.build_gather_plan(gd, g)
    ngf.LevelObjective.from_device(T, T, plan, ngf.NgfParams(), 1.0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        obj = ngf.LevelObjective.from_device(T, T, plan, ngf.NgfParams(), 1.0)
        torch.cuda.synchronize()
        del obj
    print(f"{n}^3: level setup {(time.perf_counter() - t0) / 3 * 1000:.2f} ms")
