"""H2D / D2H bandwidth probe of this box's PCIe path for the e2e staging buffers:
pinned vs write-combined vs registered vs pageable, one copy vs chunked over streams."""
import ctypes, os, sys, time
import numpy as np
import torch

torch.cuda.init()
rt = ctypes.CDLL(os.path.join(os.path.dirname(__import__("nvidia.cuda_runtime").cuda_runtime.__file__), "lib", "libcudart.so.12"))
vp = ctypes.c_void_p

def host_alloc(nb, flags):
    p = vp()
    assert rt.cudaHostAlloc(ctypes.byref(p), ctypes.c_size_t(nb), ctypes.c_uint(flags)) == 0
    return p.value

def timed(f, reps=40):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps

s = torch.cuda.current_stream().cuda_stream
for nb in (3_300_000, 13_000_000, 64_000_000):
    d = torch.empty(nb, dtype=torch.uint8, device="cuda")
    dptr = d.data_ptr()
    res = {}
    for name, flags in (("pinned", 0), ("portable", 1), ("wc", 4), ("mapped", 2)):
        h = host_alloc(nb, flags)
        ctypes.memset(h, 1, nb)
        res[name + " h2d"] = timed(lambda: rt.cudaMemcpyAsync(vp(dptr), vp(h), ctypes.c_size_t(nb), 1, vp(s)))
        res[name + " d2h"] = timed(lambda: rt.cudaMemcpyAsync(vp(h), vp(dptr), ctypes.c_size_t(nb), 2, vp(s)))
        streams = [torch.cuda.Stream() for _ in range(4)]
        def chunked(k=4):
            step = nb // k
            cur = torch.cuda.current_stream()
            for i, st in enumerate(streams[:k]):
                st.wait_stream(cur)
                rt.cudaMemcpyAsync(vp(dptr + i * step), vp(h + i * step), ctypes.c_size_t(step), 1, vp(st.cuda_stream))
            for st in streams[:k]:
                cur.wait_stream(st)
        res[name + " h2d x4 streams"] = timed(chunked)
        rt.cudaFreeHost(vp(h))
    a = np.ones(nb, np.uint8)
    res["pageable h2d"] = timed(lambda: rt.cudaMemcpyAsync(vp(dptr), vp(a.ctypes.data), ctypes.c_size_t(nb), 1, vp(s)))
    res["pageable d2h"] = timed(lambda: rt.cudaMemcpyAsync(vp(a.ctypes.data), vp(dptr), ctypes.c_size_t(nb), 2, vp(s)))
    assert rt.cudaHostRegister(vp(a.ctypes.data), ctypes.c_size_t(nb), 0) == 0
    res["registered h2d"] = timed(lambda: rt.cudaMemcpyAsync(vp(dptr), vp(a.ctypes.data), ctypes.c_size_t(nb), 1, vp(s)))
    t0 = time.perf_counter(); rt.cudaHostUnregister(vp(a.ctypes.data)); rt.cudaHostRegister(vp(a.ctypes.data), ctypes.c_size_t(nb), 0)
    res["register+unregister cost"] = time.perf_counter() - t0
    rt.cudaHostUnregister(vp(a.ctypes.data))
    for k, v in res.items():
        print(f"{nb/1e6:6.1f} MB {k:28s} {v*1e6:9.1f} us  {nb/v/1e9:6.1f} GB/s")

nb = 3_300_000
d = torch.empty(nb // 4, dtype=torch.float32, device="cuda")
hp = torch.empty(nb // 4, dtype=torch.float32, pin_memory=True)
print("torch pinned?", hp.is_pinned())
for nbk in (False, True):
    v = timed(lambda: d.copy_(hp, non_blocking=nbk))
    print(f"torch copy_ h2d non_blocking={nbk}: {v*1e6:.1f} us")
    v = timed(lambda: hp.copy_(d, non_blocking=nbk))
    print(f"torch copy_ d2h non_blocking={nbk}: {v*1e6:.1f} us")
