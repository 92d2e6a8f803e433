"""Host-buffer entry points (csrc/hostio.cu): staged uploads / downloads are byte-exact
for every size class (empty, below the direct threshold, chunked, ragged tails), page-locked
buffers take the direct path, and ngf_level_eval_host (LevelObjective.__call__ with numpy
in / out, objective.py:48-60) returns exactly what the device-resident evaluation does."""

import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_1812_06765_b200 as ngf  # noqa: E402
from paper_1812_06765_b200 import _device as dev  # noqa: E402
from paper_1812_06765_b200._lib import NGF_EARG, lib  # noqa: E402


def _stream():
    return torch.cuda.current_stream().cuda_stream


@pytest.mark.parametrize("nbytes", [0, 1, 4093, 256 << 10, (256 << 10) + 1, 3_145_731, (24 << 20) + 17])
def test_staged_round_trip(nbytes):
    rng = np.random.default_rng(nbytes)
    src = rng.integers(0, 256, nbytes, dtype=np.uint8)
    d = torch.empty(max(nbytes, 1), dtype=torch.uint8, device="cuda")
    assert lib().ngf_host_upload(d.data_ptr(), src.ctypes.data, nbytes, _stream()) == 0
    src_copy = src.copy()
    src[:] = 0  # the source may be reused as soon as the call returns
    back = np.full(nbytes, 7, np.uint8)
    assert lib().ngf_host_download(back.ctypes.data, d.data_ptr(), nbytes, _stream()) == 0
    assert np.array_equal(back, src_copy)
    if nbytes:
        assert np.array_equal(d[:nbytes].cpu().numpy(), src_copy)


def test_pinned_direct_and_args():
    x = torch.arange(1 << 20, dtype=torch.float32).pin_memory()
    d = torch.empty_like(x, device="cuda")
    assert lib().ngf_host_upload(d.data_ptr(), x.data_ptr(), x.numel() * 4, _stream()) == 0
    out = torch.empty_like(x).pin_memory()
    assert lib().ngf_host_download(out.data_ptr(), d.data_ptr(), x.numel() * 4, _stream()) == 0
    assert torch.equal(out, x)
    assert lib().ngf_host_upload(None, x.data_ptr(), 4, _stream()) == NGF_EARG
    assert lib().ngf_host_download(out.data_ptr(), None, 4, _stream()) == NGF_EARG


def test_to_device_to_host_large():
    a = np.random.default_rng(0).standard_normal((3, 70, 66, 65)).astype(np.float32)
    t = dev.to_device(a)
    assert np.array_equal(t.cpu().numpy(), a)
    assert np.array_equal(dev.to_host(t), a)


@pytest.mark.parametrize("exact", [False, True])
def test_eval_host_matches_device(exact):
    R, T, _ = ngf.ct_pair(48, dtype=np.float32)
    gd = ngf.deformation_grid_for(R.grid, 4)
    plan = ngf.build_gather_plan(gd, R.grid)
    obj = ngf.LevelObjective.from_device(torch.from_numpy(T.values).cuda(), torch.from_numpy(R.values).cuda(),
                                         plan, ngf.NgfParams(10.0, 10.0), 1.0, exact=exact)
    y = ngf.smooth_random_field(gd, seed=3, amplitude_mm=2.0).field.astype(np.float32).ravel()
    xd = torch.from_numpy(y).cuda()
    gdv = torch.empty_like(xd)
    sc = obj.eval_device(xd, gdv).cpu().numpy()
    for x in (y, torch.from_numpy(y).pin_memory().numpy(), y.astype(np.float64)):
        J, g = obj(x)
        assert J == float(sc[0]) and obj.last_D == float(sc[1]) and obj.last_S == float(sc[2])
        assert g.dtype == np.float32 and np.array_equal(g, gdv.cpu().numpy())
    with pytest.raises(ValueError):
        obj(y[:-3])
    # direct C-ABI call with a pageable output buffer (staged download)
    g2 = np.empty_like(y)
    s3 = (ctypes.c_double * 3)()
    assert lib().ngf_level_eval_host(obj.level.handle, y.ctypes.data, g2.ctypes.data,
                                     ctypes.cast(s3, ctypes.c_void_p), 1 if exact else 0, _stream()) == 0
    assert list(s3) == [float(v) for v in sc] and np.array_equal(g2, gdv.cpu().numpy())
    assert lib().ngf_level_eval_host(obj.level.handle, y.ctypes.data, g2.ctypes.data,
                                     ctypes.cast(s3, ctypes.c_void_p), 3, _stream()) == NGF_EARG
