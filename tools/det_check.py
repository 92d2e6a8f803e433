"""Bit-determinism of the fused evaluation: repeated evaluations, alone and with other
streams busy (python tools/det_check.py n ratio)."""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1812_06765_b200 as ngf  # noqa: E402

n, ratio = int(sys.argv[1]), int(sys.argv[2])
objs = []
for seed in range(3):
    R, T, gd, y, _ = bench.make_inputs(n, ratio, seed=seed)
    obj = ngf.LevelObjective.from_device(torch.from_numpy(T.values).cuda(), torch.from_numpy(R.values).cuda(),
                                         ngf.build_gather_plan(gd, R.grid), ngf.NgfParams(10.0, 10.0), 1.0)
    objs.append((obj, torch.from_numpy(y.ravel().copy()).cuda()))


def run(i, reps, out, stream=None):
    obj, x = objs[i]
    g = torch.empty_like(x)
    res = []
    ctx = torch.cuda.stream(stream) if stream is not None else torch.cuda.stream(torch.cuda.current_stream())
    with ctx:
        for _ in range(reps):
            sc = obj.eval_device(x, g)
            res.append((float(sc[0].item()), g.cpu().numpy().copy()))
    out[i] = res


base = {}
run(0, 1, base)
J0, g0 = base[0][0]
out = {}
run(0, 20, out)
print("alone: all identical", all(J == J0 and np.array_equal(g, g0) for J, g in out[0]))
streams = [torch.cuda.Stream() for _ in range(3)]
out = {}
th = [threading.Thread(target=run, args=(i, 20, out, streams[i])) for i in range(3)]
for t in th:
    t.start()
for t in th:
    t.join()
ok = [J == J0 and np.array_equal(g, g0) for J, g in out[0]]
print("concurrent: identical", sum(ok), "of", len(ok))
if not all(ok):
    J, g = out[0][ok.index(False)]
    d = np.abs(g - g0)
    print("  J", J, J0, "max grad diff", d.max(), "at", np.unravel_index(d.argmax(), g.shape), "n diff", int((d > 0).sum()))
