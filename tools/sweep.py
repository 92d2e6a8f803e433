"""Time the fused kernel per variant / z-chunk at one size (CUDA events inside the library).

    python tools/sweep.py [--n 256] [--variants 0,1,2,3] [--cz 0]
"""

import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_06765_b200 as ngf  # noqa: E402
from paper_1812_06765_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--ratio", type=int, default=4)
    ap.add_argument("--variants", default="0,1,2,3")
    ap.add_argument("--cz", default="0")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    R, T, _ = ngf.ct_pair(a.n, dtype=np.float32)
    gd = ngf.deformation_grid_for(R.grid, a.ratio)
    y = ngf.smooth_random_field(gd, seed=2, amplitude_mm=2.0).field.astype(np.float32)
    plan = ngf.build_gather_plan(gd, R.grid)
    Td, Rd = torch.from_numpy(T.values).cuda(), torch.from_numpy(R.values).cuda()
    x = torch.from_numpy(y.ravel().copy()).cuda()
    g = torch.empty_like(x)
    ref = None
    N = R.grid.num_points
    for v in [int(s) for s in a.variants.split(",")]:
        for cz in [int(s) for s in a.cz.split(",")]:
            os.environ["NGF_FUSED_VARIANT"] = str(v)
            if cz:
                os.environ["NGF_FUSED_CZ"] = str(cz)
            else:
                os.environ.pop("NGF_FUSED_CZ", None)
            obj = ngf.LevelObjective.from_device(Td, Rd, plan, ngf.NgfParams(), 1.0)
            lv = obj.level
            _lib.check(_lib.lib().ngf_level_set_timing(lv.handle, 1), "timing")
            for _ in range(3):
                obj.eval_device(x, g)
            ms = []
            for _ in range(a.reps):
                obj.eval_device(x, g)
                t = ctypes.c_float()
                _lib.check(_lib.lib().ngf_level_kernel_ms(lv.handle, ctypes.byref(t)), "ms")
                ms.append(t.value)
            info = (ctypes.c_int64 * 9)()
            _lib.lib().ngf_level_info(lv.handle, info)
            gh = g.cpu().numpy()
            if ref is None:
                ref = gh
            rel = np.linalg.norm(gh - ref) / np.linalg.norm(ref)
            med = float(np.median(ms))
            gbs = (20 * N + 12 * gd.num_points) / (med / 1e3) / 1e9
            print(f"variant {v} cz {info[2]:3d} ctas {info[0]:5d} smem {info[1]:6d}: kernel {med:.3f} ms "
                  f"(min {min(ms):.3f}) {gbs:7.1f} GB/s  grad-vs-first {rel:.1e}", flush=True)
            del obj, lv


if __name__ == "__main__":
    main()
