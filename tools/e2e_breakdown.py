"""Break the numpy-facing evaluation (LevelObjective.__call__ -> ngf_level_eval_host) at
256^3 / 64^3 f32 into its host and device parts.  On a B200: python tools/e2e_breakdown.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1812_06765_b200 as ngf  # noqa: E402
from paper_1812_06765_b200._lib import lib  # noqa: E402

R, T, gd, y, _ = bench.make_inputs(256, 4, seed=0)
obj = ngf.LevelObjective.from_device(torch.from_numpy(T.values).cuda(), torch.from_numpy(R.values).cuda(),
                                     ngf.build_gather_plan(gd, R.grid), ngf.NgfParams(10.0, 10.0), 1.0)
xh = y.ravel().copy()
n = xh.size
for _ in range(5):
    obj(xh)
torch.cuda.synchronize()
s = torch.cuda.current_stream().cuda_stream


def timeit(name, f, reps=100):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    print(f"{name:44s} {(time.perf_counter() - t0) / reps * 1e6:9.1f} us")


x_dev = torch.empty(n, device="cuda")
g_dev = torch.empty(n, device="cuda")
sc_dev = torch.zeros(3, dtype=torch.float64, device="cuda")
g_pin = torch.empty(n, pin_memory=True)
g_np = np.empty(n, np.float32)
x_pin = torch.from_numpy(xh).pin_memory()
timeit("full __call__ (numpy in, pinned numpy out)", lambda: obj(xh))
timeit("staged upload 3.1 MB (pageable src)", lambda: lib().ngf_host_upload(x_dev.data_ptr(), xh.ctypes.data, xh.nbytes, s))
timeit("direct upload 3.1 MB (pinned src)", lambda: lib().ngf_host_upload(x_dev.data_ptr(), x_pin.data_ptr(), xh.nbytes, s))
timeit("eval_device", lambda: obj.eval_device(x_dev, g_dev, sc_dev))
timeit("download 3.1 MB to pinned (+sync)", lambda: lib().ngf_host_download(g_pin.data_ptr(), g_dev.data_ptr(), xh.nbytes, s))
timeit("staged download 3.1 MB to pageable", lambda: lib().ngf_host_download(g_np.ctypes.data, g_dev.data_ptr(), xh.nbytes, s))
timeit("torch pageable H2D", lambda: x_dev.copy_(torch.from_numpy(xh)))
timeit("numpy memcpy 3.1 MB", lambda: g_np.__setitem__(slice(None), xh))
big = np.ones(64 << 20, np.uint8)
bd = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
timeit("staged upload 64 MB", lambda: lib().ngf_host_upload(bd.data_ptr(), big.ctypes.data, big.nbytes, s), 20)
timeit("staged download 64 MB", lambda: lib().ngf_host_download(big.ctypes.data, bd.data_ptr(), big.nbytes, s), 20)
timeit("torch pageable H2D 64 MB", lambda: bd.copy_(torch.from_numpy(big)), 20)
timeit("torch pageable D2H 64 MB", lambda: torch.from_numpy(big).copy_(bd), 20)
g0 = obj(xh)[1].copy()
xd = torch.from_numpy(xh).cuda()
gd_ = torch.empty_like(xd)
obj.eval_device(xd, gd_)
print("host call == device call:", np.array_equal(g0, gd_.cpu().numpy()))

# A/B against the torch-staged call this replaced (single-thread memcpy into a pinned
# buffer, torch H2D, eval, torch D2H into a fresh pinned buffer)
xp = torch.empty(n, pin_memory=True)
scp = torch.empty(3, dtype=torch.float64, pin_memory=True)


def torch_staged():
    xp.numpy()[:] = xh
    x_dev.copy_(xp, non_blocking=True)
    obj.eval_device(x_dev, g_dev, sc_dev)
    go = torch.empty(n, pin_memory=True)
    go.copy_(g_dev, non_blocking=True)
    scp.copy_(sc_dev, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return go


for rep in range(3):
    timeit(f"[{rep}] ngf_level_eval_host call", lambda: obj(xh), 300)
    timeit(f"[{rep}] torch-staged call", torch_staged, 300)
