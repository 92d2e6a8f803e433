"""One traced pipelined host evaluation per part count (NGF_PIPE_TRACE=1 prints the
event times of every stage): python tools/pipe_trace.py [n] [ratio]"""
import os
import sys

os.environ["NGF_PIPE_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
for parts in (2, 3, 4, 5, 8):
    lib().ngf_level_set_host_pipeline(obj.level.handle, parts)
    for _ in range(4):
        obj(yp.numpy())
    sys.stderr.flush()
