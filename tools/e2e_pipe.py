"""Per-call time of the numpy-facing evaluation (page-locked y and gradient) for each
part count of the pipelined host evaluation (ngf_level_set_host_pipeline), against the
device-resident evaluation.  On a B200: python tools/e2e_pipe.py [n] [ratio]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1812_06765_b200 as ngf  # noqa: E402
from paper_1812_06765_b200._lib import lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ratio = int(sys.argv[2]) if len(sys.argv) > 2 else 4
R, T, gd, y, _ = bench.make_inputs(n, ratio, seed=0)
obj = ngf.LevelObjective.from_device(torch.from_numpy(T.values).cuda(), torch.from_numpy(R.values).cuda(),
                                     ngf.build_gather_plan(gd, R.grid), ngf.NgfParams(10.0, 10.0), 1.0)
yp = torch.empty(y.size, dtype=torch.float32, pin_memory=True)
yp.numpy()[:] = y.ravel()
x = yp.cuda()
g = torch.empty_like(x)
sc = torch.zeros(3, dtype=torch.float64, device="cuda")
for _ in range(5):
    obj.eval_device(x, g, sc)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    obj.eval_device(x, g, sc)
e1.record()
torch.cuda.synchronize()
print(f"{n}^3 r{ratio}: device-resident eval {e0.elapsed_time(e1) / 50 * 1e3:.1f} us")
for rep in range(2):
    for parts in (1, 2, 3, 4, 5, 6, 8):
        lib().ngf_level_set_host_pipeline(obj.level.handle, parts)
        for _ in range(5):
            obj(yp.numpy())
        t0 = time.perf_counter()
        for _ in range(100):
            obj(yp.numpy())
        dt = (time.perf_counter() - t0) / 100
        print(f"  parts {parts}: {dt * 1e6:.1f} us per call = {1 / dt:.0f} evals/s")
