"""Cost of pinning a pageable numpy buffer in place (cudaHostRegister) + a direct DMA, vs
the staged upload (ngf_host_upload) and a pageable cudaMemcpy, for 64 MB and 3 MB.
On a B200: python tools/host_register_probe.py"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1812_06765_b200._lib import lib  # noqa: E402

rt = ctypes.CDLL("libcudart.so.12") if False else None
cudart = torch.cuda.cudart()
s = torch.cuda.current_stream().cuda_stream


def t(f, reps=10):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


for mb in (64, 3):
    n = mb << 20
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for fresh in (False, True):
        a = np.ones(n, np.uint8)

        def reg_copy():
            # a fresh array each time when `fresh` (pages never pinned before)
            b = np.ones(n, np.uint8) if fresh else a
            p = b.ctypes.data
            r = cudart.cudaHostRegister(p, n, 0)
            assert int(r) == 0, r
            d.copy_(torch.from_numpy(b), non_blocking=True)
            torch.cuda.synchronize()
            cudart.cudaHostUnregister(p)

        def staged():
            b = np.ones(n, np.uint8) if fresh else a
            lib().ngf_host_upload(d.data_ptr(), b.ctypes.data, n, s)

        def plain():
            b = np.ones(n, np.uint8) if fresh else a
            d.copy_(torch.from_numpy(b))

        def alloc_only():
            np.ones(n, np.uint8)

        base = t(alloc_only) if fresh else 0.0
        print(f"{mb} MB {'fresh' if fresh else 'reused'} buffer: register+DMA+unregister {t(reg_copy) - base:.3f} ms, "
              f"staged {t(staged) - base:.3f} ms, pageable cudaMemcpy {t(plain) - base:.3f} ms"
              + (f" (allocation {base:.3f} ms subtracted)" if fresh else ""))
