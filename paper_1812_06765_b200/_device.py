"""Device plumbing: torch is used only for CUDA memory and streams.

Every compute call goes through libngfb200.so; these helpers just move numpy
arrays to/from CUDA tensors and hand raw pointers and the current stream to
the C-ABI.  A missing CUDA device is an error, never a silent CPU path.
"""

from __future__ import annotations

import numpy as np

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as _t
        _torch = _t
    return _torch


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("paper_1812_06765_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return t


def torch_dtype(dtype):
    t = torch()
    if isinstance(dtype, t.dtype):
        return dtype
    dt = np.dtype(dtype)
    if dt == np.float32:
        return t.float32
    if dt == np.float64:
        return t.float64
    raise ValueError(f"unsupported dtype {dt}")


def np_dtype(tdtype):
    t = torch()
    return np.float32 if tdtype == t.float32 else np.float64


def is_tensor(v) -> bool:
    return type(v).__module__.startswith("torch")


def to_device(a, dtype=None):
    """numpy array or tensor -> contiguous CUDA tensor (dtype preserved unless given)."""
    t = require_cuda()
    if is_tensor(a):
        out = a
        if dtype is not None:
            out = out.to(torch_dtype(dtype))
        if not out.is_cuda:
            out = out.cuda()
        return out.contiguous()
    arr = np.ascontiguousarray(a if dtype is None else np.asarray(a).astype(dtype, copy=False))
    if arr.nbytes >= _BIG_UPLOAD and arr.dtype in (np.float32, np.float64):
        return _upload_pinned(t, arr)
    return t.from_numpy(arr).cuda()


# Large host arrays (volumes) go through a reusable page-locked staging buffer filled by a
# few threads (numpy copies release the GIL), then one asynchronous DMA: ~2x the
# bandwidth of a pageable copy (measured 4 ms vs 6-8 ms for a 256^3 f32 volume).
_BIG_UPLOAD = 8 << 20
_stage = {"buf": None, "event": None, "pool": None}


def par_copy(dst: np.ndarray, src: np.ndarray, parts: int = 4) -> None:
    """dst[...] = src with a few threads (numpy copies release the GIL): host staging
    copies of multi-MB vectors run at ~4x the single-thread bandwidth."""
    d, s = dst.reshape(-1), src.reshape(-1)
    if s.nbytes < (1 << 20):
        d[:] = s
        return
    st = _stage
    if st["pool"] is None:
        from concurrent.futures import ThreadPoolExecutor

        st["pool"] = ThreadPoolExecutor(4)
    step = (s.size + parts - 1) // parts
    list(st["pool"].map(lambda i: np.copyto(d[i * step:(i + 1) * step], s[i * step:(i + 1) * step]),
                        range(parts)))


def _upload_pinned(t, arr: np.ndarray):
    st = _stage
    if st["buf"] is None or st["buf"].numel() < arr.nbytes:
        if st["event"] is not None:
            st["event"].synchronize()
        st["buf"] = t.empty(arr.nbytes, dtype=t.uint8, pin_memory=True)
        st["event"] = None
    if st["event"] is not None:
        st["event"].synchronize()  # the previous upload has left the staging buffer
    stage = st["buf"][: arr.nbytes].numpy().view(arr.dtype).reshape(arr.shape)
    par_copy(stage, arr)
    out = t.empty(arr.shape, dtype=torch_dtype(arr.dtype), device="cuda")
    out.view(-1).view(t.uint8).copy_(st["buf"][: arr.nbytes], non_blocking=True)
    ev = t.cuda.Event()
    ev.record()
    st["event"] = ev
    return out


def empty(shape, dtype):
    t = require_cuda()
    return t.empty(tuple(shape), dtype=torch_dtype(dtype), device="cuda")


def zeros(shape, dtype):
    t = require_cuda()
    return t.zeros(tuple(shape), dtype=torch_dtype(dtype), device="cuda")


def ptr(x) -> int:
    return int(x.data_ptr()) if x is not None else 0


def stream() -> int:
    return int(torch().cuda.current_stream().cuda_stream)


def to_host(x) -> np.ndarray:
    return x.detach().cpu().numpy()


def synchronize() -> None:
    """Wait for the current stream's work (host-side timing of device calls)."""
    torch().cuda.current_stream().synchronize()
