"""One fused evaluation per shape, for compute-sanitizer (racecheck / initcheck / memcheck):
    compute-sanitizer --tool racecheck python tools/sanitize_lean.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1812_06765_b200 as ngf  # noqa: E402

for dims, ratio in (((64, 64, 64), 4), ((64, 64, 64), 2), ((33, 97, 18), 2), ((130, 20, 150), 4)):
    gi = ngf.Grid3(dims, (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    gd = ngf.deformation_grid_for(gi, ratio)
    R = ngf.smooth_random_volume(gi, seed=5).values.astype(np.float32)
    T = ngf.smooth_random_volume(gi, seed=6).values.astype(np.float32)
    y = ngf.smooth_random_field(gd, seed=7, amplitude_mm=4.0).field.astype(np.float32)
    obj = ngf.LevelObjective.from_device(torch.from_numpy(T).cuda(), torch.from_numpy(R).cuda(),
                                         ngf.build_gather_plan(gd, gi), ngf.NgfParams(), 1.0)
    x = torch.from_numpy(y.ravel().copy()).cuda()
    g = torch.empty_like(x)
    sc = obj.eval_device(x, g)
    torch.cuda.synchronize()
    print(dims, ratio, float(sc[0].item()), flush=True)
