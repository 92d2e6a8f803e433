"""A/B of fused-march variants at one configuration: kernel time (CUDA events on the
launching stream, mean of N after warm-up) and whole-evaluation time.

    python tools/variant_ab.py [n] [ratio] [variants...]      (default 256 4 6 2)
"""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_06765_b200 as ngf  # noqa: E402
from paper_1812_06765_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ratio = int(sys.argv[2]) if len(sys.argv) > 2 else 4
variants = [int(v) for v in sys.argv[3:]] or [6, 2]
R, T, _ = ngf.ct_pair(n, seed=0)
gd = ngf.deformation_grid_for(R.grid, ratio)
y = ngf.smooth_random_field(gd, seed=2, amplitude_mm=2.0).field.astype(np.float32)
T_dev, R_dev = torch.from_numpy(T.values).cuda(), torch.from_numpy(R.values).cuda()
x = torch.from_numpy(y.ravel().copy()).cuda()
ref = None
for rep in range(2):
    for v in variants:
        os.environ["NGF_FUSED_VARIANT"] = str(v)
        obj = ngf.LevelObjective.from_device(T_dev, R_dev, ngf.build_gather_plan(gd, R.grid), ngf.NgfParams(), 1.0)
        lvl = obj.level
        g = torch.empty_like(x)
        sc = torch.zeros(3, dtype=torch.float64, device="cuda")
        for _ in range(5):
            obj.eval_device(x, g, sc)
        torch.cuda.synchronize()
        _lib.lib().ngf_level_set_timing(lvl.handle, 1)
        ks = []
        for _ in range(30):
            obj.eval_device(x, g, sc)
            ms = ctypes.c_float()
            _lib.lib().ngf_level_kernel_ms(lvl.handle, ctypes.byref(ms))
            ks.append(ms.value)
        _lib.lib().ngf_level_set_timing(lvl.handle, 0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            obj.eval_device(x, g, sc)
        e1.record()
        torch.cuda.synchronize()
        info = (ctypes.c_int64 * 9)()
        _lib.lib().ngf_level_info(lvl.handle, info)
        J = float(sc[0].item())
        gh = g.cpu().numpy()
        if ref is None:
            ref = (J, gh)
        dJ = abs(J - ref[0]) / abs(ref[0])
        dg = float(np.linalg.norm(gh - ref[1]) / np.linalg.norm(ref[1]))
        print(f"{n}^3 r{ratio} variant {_lib.lib().ngf_level_variant(lvl.handle)}: kernel {np.mean(ks)*1e3:.1f} us "
              f"(min {np.min(ks)*1e3:.1f}), eval {e0.elapsed_time(e1) / 50 * 1e3:.1f} us, ctas {info[0]}, "
              f"smem {info[1]}, cz {info[2]}, J {J:.9g} (vs first {dJ:.1e}), grad vs first {dg:.1e}", flush=True)
        del obj, lvl
