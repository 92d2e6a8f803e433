"""Registration determinism: sequential repeats and concurrent streams vs sequential
(the concurrency test of tests/test_gpu_register.py, with diagnostics)."""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1812_06765_b200 as ngf  # noqa: E402

cfg = ngf.MultilevelConfig(num_levels=3, grid_ratio=4, precision="f32", lbfgs=ngf.LbfgsConfig(max_iterations=8))
pairs = [ngf.ct_pair(128, seed=500 + p, dtype=np.float32)[:2] for p in range(6)]
ref = [ngf.register(R, T, cfg) for R, T in pairs]
ref2 = [ngf.register(R, T, cfg) for R, T in pairs]
print("sequential repeat identical:", [np.array_equal(a[0].field, b[0].field) for a, b in zip(ref, ref2)])
# one registration on a user stream, alone
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    one = ngf.register(*pairs[0], cfg)
    s.synchronize()
print("user stream alone identical:", np.array_equal(one[0].field, ref[0][0].field))
lv_ref = [(lv.iterations, lv.evaluations, [r.J for r in lv.records]) for lv in ref[0][1].levels]
lv_one = [(lv.iterations, lv.evaluations, [r.J for r in lv.records]) for lv in one[1].levels]
for a, b in zip(lv_ref, lv_one):
    if a != b:
        print("  first differing level: ref", a[0], a[1], a[2][:4], "stream", b[0], b[1], b[2][:4])
        break
