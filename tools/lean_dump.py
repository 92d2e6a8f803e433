"""Evaluate the fused objective once and save (J, grad) (A/B of build or env variants of
the lean march): python tools/lean_dump.py n ratio out.npz"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1812_06765_b200 as ngf  # noqa: E402

n, ratio, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
R, T, gd, y, _ = bench.make_inputs(n, ratio, seed=0)
obj = ngf.LevelObjective.from_device(torch.from_numpy(T.values).cuda(), torch.from_numpy(R.values).cuda(),
                                     ngf.build_gather_plan(gd, R.grid), ngf.NgfParams(10.0, 10.0), 1.0)
x = torch.from_numpy(y.ravel().copy()).cuda()
g = torch.empty_like(x)
sc = obj.eval_device(x, g)
np.savez(out, J=float(sc[0].item()), g=g.cpu().numpy())
