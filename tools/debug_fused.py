"""Locate disagreements between the fused and the exact evaluation on one shape."""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_06765_b200 as ngf  # noqa: E402


def run(dims, ratio, spacing=(1.0, 1.1, 0.9)):
    gi = ngf.Grid3(dims, spacing, (-3.0, 2.0, 1.0))
    gd = ngf.deformation_grid_for(gi, ratio)
    R = ngf.smooth_random_volume(gi, seed=5).values.astype(np.float32)
    T = ngf.smooth_random_volume(gi, seed=6).values.astype(np.float32)
    y = ngf.smooth_random_field(gd, seed=7, amplitude_mm=2.5).field.astype(np.float32)
    plan = ngf.build_gather_plan(gd, gi)
    Td, Rd = torch.from_numpy(T).cuda(), torch.from_numpy(R).cuda()
    f = ngf.LevelObjective.from_device(Td, Rd, plan, ngf.NgfParams(), 1.0)
    e = ngf.LevelObjective.from_device(Td, Rd, plan, ngf.NgfParams(), 1.0, exact=True)
    J1, g1 = f(y.ravel())
    J2, g2 = e(y.ravel())
    info = (__import__("ctypes").c_int64 * 9)()
    ngf._lib.lib().ngf_level_info(f.level.handle, info)
    g1 = g1.reshape((3,) + gd.shape)
    g2 = g2.reshape((3,) + gd.shape)
    d = np.abs(g1 - g2)
    rel = np.linalg.norm(g1 - g2) / np.linalg.norm(g2)
    print(f"dims {dims} ratio {ratio} cz {info[2]} win {info[3]},{info[4]},{info[5]} tiles "
          f"{info[6]},{info[7]},{info[8]}: J {J1:.7g} vs {J2:.7g}; grad rel {rel:.3e}")
    if rel > 1e-4:
        bad = np.argwhere(d > 1e-3 * np.abs(g2).max())
        print("  bad nodes (c,z,y,x) sample:", bad[:10].tolist(), "count", len(bad))
        for ax, name in ((1, "z"), (2, "y"), (3, "x")):
            prof = d.max(axis=tuple(a for a in range(4) if a != ax))
            print(f"  max err along {name}:", np.round(prof / np.abs(g2).max(), 4).tolist())


if __name__ == "__main__":
    for cz in (None, "1", "2", "4", "8"):
        if cz:
            os.environ["NGF_FUSED_CZ"] = cz
        run((40, 40, 40), 1)
    os.environ.pop("NGF_FUSED_CZ", None)
    run((40, 40, 40), 2)
    run((64, 64, 64), 4)
