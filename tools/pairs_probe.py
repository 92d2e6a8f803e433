"""Config 4 on one GPU: registrations in flight on K host threads / CUDA streams; pairs/s
and a bitwise comparison of every field with the sequential run.

    python tools/pairs_probe.py [--pairs 16] [--n 256]
    SCHED=1|2|4 python tools/pairs_probe.py ...   # context scheduling: spin / yield / blocking sync
"""
import argparse
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("SCHED"):  # cudaDeviceScheduleSpin 1 / Yield 2 / BlockingSync 4, before the context exists
    import ctypes
    import glob
    import torch as _t  # noqa: F401  (loads torch's cudart)
    import nvidia
    _cr = glob.glob(os.path.join(nvidia.__path__[0], "cuda_runtime", "lib", "libcudart.so*"))
    _rt = ctypes.CDLL(_cr[0] if _cr else "libcudart.so.12")
    print("cudaSetDeviceFlags", int(os.environ["SCHED"]), "->", _rt.cudaSetDeviceFlags(int(os.environ["SCHED"])))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1812_06765_b200 as ngf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--pairs", type=int, default=16)
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--streams", default="1,2,3,4,6,8")
ap.add_argument("--levels", type=int, default=4)
a = ap.parse_args()
cfg = ngf.MultilevelConfig(num_levels=a.levels, grid_ratio=4, precision="f32")
batch = [bench.make_inputs(a.n, 4, seed=1000 + p)[:2] for p in range(a.pairs)]
ngf.register(*batch[0], cfg)
ref = [ngf.register(R, T, cfg)[0].field for R, T in batch]


def run(k):
    streams = [torch.cuda.Stream() for _ in range(k)]
    for st in streams:  # warm: reduction scratch and torch's block cache of each stream
        with torch.cuda.stream(st):
            ngf.register(*batch[0], cfg)
        st.synchronize()
    out = [None] * len(batch)
    per = [0.0] * k

    def work(i):
        t0 = time.perf_counter()
        with torch.cuda.stream(streams[i]):
            for j in range(i, len(batch), k):
                out[j] = ngf.register(*batch[j], cfg)[0].field
            streams[i].synchronize()
        per[i] = time.perf_counter() - t0

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    th = [threading.Thread(target=work, args=(i,)) for i in range(k)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    same = all(np.array_equal(o, r) for o, r in zip(out, ref))
    print(f"streams {k}: {len(batch) / dt:6.1f} pairs/s ({dt:.3f} s; per thread "
          f"{', '.join(f'{p:.3f}' for p in per)}); fields bit-identical to sequential: {same}", flush=True)


for k in (int(v) for v in a.streams.split(",")):
    run(k)
