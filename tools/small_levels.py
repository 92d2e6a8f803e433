"""Device time of one evaluation and one L-BFGS two-loop at the coarse pyramid levels
(32^3/8^3 .. 128^3/32^3), CUDA events, back-to-back launches.

    python tools/small_levels.py            # timings
    ncu --metrics gpu__time_duration.sum --clock-control none python tools/small_levels.py --once
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1812_06765_b200 as ngf  # noqa: E402
from paper_1812_06765_b200._lib import lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--once", action="store_true")
a = ap.parse_args()
reps = 1 if a.once else 200
s = torch.cuda.current_stream()
for n in (32, 64, 128, 256):
    R, T, gd, y, _ = bench.make_inputs(n, 4, seed=0)
    obj = ngf.LevelObjective.from_device(torch.from_numpy(T.values).cuda(), torch.from_numpy(R.values).cuda(),
                                         ngf.build_gather_plan(gd, R.grid), ngf.NgfParams(10.0, 10.0), 1.0)
    x = torch.from_numpy(y.ravel().copy()).cuda()
    g = torch.empty_like(x)
    sc = torch.zeros(3, dtype=torch.float64, device="cuda")
    info = (ctypes.c_int64 * 9)()
    lib().ngf_level_info(obj.level.handle, info)
    m = 10
    S = [torch.randn_like(x) for _ in range(m)]
    Y = [torch.randn_like(x) for _ in range(m)]
    Sp = (ctypes.c_void_p * m)(*[t.data_ptr() for t in S])
    Yp = (ctypes.c_void_p * m)(*[t.data_ptr() for t in Y])
    rho = (ctypes.c_double * m)(*([0.01] * m))
    d = torch.empty_like(x)
    slope = torch.zeros(1, dtype=torch.float64, device="cuda")
    res = {}
    for name, f in (("eval", lambda: obj.eval_device(x, g, sc)),
                    ("two_loop m=10", lambda: lib().ngf_lbfgs_two_loop(0, Sp, Yp, rho, ctypes.c_double(1.0), m,
                                                                       g.data_ptr(), d.data_ptr(), x.numel(),
                                                                       slope.data_ptr(), s.cuda_stream))):
        f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            f()
        e1.record()
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / reps * 1e3
    print(f"{n}^3 / {gd.dims[0]}^3: ctas {info[0]} cz {info[2]} " +
          "  ".join(f"{k} {v:.1f} us" for k, v in res.items()))
