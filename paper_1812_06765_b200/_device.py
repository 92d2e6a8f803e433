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
    if arr.nbytes >= _BIG and arr.dtype in (np.float32, np.float64):
        return _upload_staged(t, arr)
    return t.from_numpy(arr).cuda()


# Large host arrays (volumes, fields) move through the library's staged transfers
# (ngf_host_upload / ngf_host_download, csrc/hostio.cu): chunked copies into page-locked
# memory on several host threads, overlapped with the DMA.  A pageable torch copy runs at
# 7-17 GB/s on the B200 boxes, the staged one near the ~50 GB/s of the link.
_BIG = 1 << 20


# Page-locked sources are uploaded by a direct, asynchronous DMA: the call returns before
# the copy engine has read the buffer.  Each such source is kept alive here until an event
# recorded after its DMA has completed, so dropping the array (and torch's host allocator
# recycling the block) cannot race the copy.  Contract: the caller must not WRITE to a
# page-locked source until the stream has passed the upload (pageable sources are copied
# into the library's staging buffer before ngf_host_upload returns, so they are free at once).
_inflight = []


def _retire_uploads():
    while _inflight and _inflight[0][0].query():
        _inflight.pop(0)


def _upload_staged(t, arr: np.ndarray):
    from ._lib import check, lib

    out = t.empty(arr.shape, dtype=torch_dtype(arr.dtype), device="cuda")
    check(lib().ngf_host_upload(out.data_ptr(), arr.ctypes.data, arr.nbytes, stream()), "ngf_host_upload")
    _retire_uploads()
    if lib().ngf_host_is_pinned(arr.ctypes.data):
        ev = t.cuda.Event()
        ev.record(t.cuda.current_stream())
        _inflight.append((ev, arr))
    return out


def pinned_empty(shape, dtype) -> np.ndarray:
    """A numpy array in page-locked host memory (torch's caching host allocator) when a GPU
    is present, so its uploads are direct DMAs; plain numpy memory otherwise."""
    t = torch()
    if t.cuda.is_available():
        return t.empty(tuple(shape), dtype=torch_dtype(dtype), pin_memory=True).numpy()
    return np.empty(shape, dtype)


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
    x = x.detach()
    if x.is_cuda and x.numel() * x.element_size() >= _BIG and x.dtype in (torch().float32, torch().float64):
        from ._lib import check, lib

        x = x.contiguous()
        out = np.empty(tuple(x.shape), dtype=np_dtype(x.dtype))
        check(lib().ngf_host_download(out.ctypes.data, x.data_ptr(), out.nbytes, stream()),
              "ngf_host_download")
        return out
    return x.cpu().numpy()


def synchronize() -> None:
    """Wait for the current stream's work (host-side timing of device calls)."""
    torch().cuda.current_stream().synchronize()
