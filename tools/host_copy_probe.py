"""Host copy bandwidth on the GPU box: staged upload vs copy-thread count."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
code = r'''
import os, time, numpy as np, torch
from paper_1812_06765_b200._lib import lib
s = torch.cuda.current_stream().cuda_stream
for nb in (3_145_728, 16 << 20, 64 << 20):
    a = np.ones(nb, np.uint8); d = torch.empty(nb, dtype=torch.uint8, device="cuda"); b = np.empty_like(a)
    def tm(f, reps):
        f(); torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(reps): f()
        torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps
    reps = 50 if nb < (8 << 20) else 10
    up = tm(lambda: lib().ngf_host_upload(d.data_ptr(), a.ctypes.data, nb, s), reps)
    dn = tm(lambda: lib().ngf_host_download(b.ctypes.data, d.data_ptr(), nb, s), reps)
    mc = tm(lambda: np.copyto(b, a), reps)
    print(f"threads={os.environ.get('NGF_HOST_THREADS')} {nb/2**20:5.1f} MiB up {up*1e6:8.1f} us ({nb/up/1e9:5.1f} GB/s) down {dn*1e6:8.1f} us ({nb/dn/1e9:5.1f} GB/s) memcpy {mc*1e6:8.1f} us ({nb/mc/1e9:5.1f} GB/s)")
'''
for k in (1, 2, 4, 8, 12):
    subprocess.run([sys.executable, "-c", code], env=dict(os.environ, NGF_HOST_THREADS=str(k)), check=True)
