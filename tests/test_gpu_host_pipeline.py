"""The pipelined numpy-facing evaluation (ngf_level_eval_host with page-locked y and
gradient: the z chunks run as groups on their own streams, uploads and downloads overlap
the march) against the serial call and the device-resident evaluation: J and the
gradient bit-identical for every part count, including a non-finite trial point
(objective.py:55-57: J = inf) and a pageable y (serial fallback)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_1812_06765_b200 as ngf  # noqa: E402
from paper_1812_06765_b200._lib import lib  # noqa: E402

CASES = [
    # (image dims, grid ratio)
    ((256, 256, 256), 4),
    ((128, 128, 128), 2),
    ((128, 128, 128), 4),
    ((96, 80, 130), 4),
    ((64, 64, 64), 4),
]


def _setup(dims, ratio, seed=0):
    gi = ngf.Grid3(dims, (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    gd = ngf.deformation_grid_for(gi, ratio)
    R = ngf.smooth_random_volume(gi, seed=seed).values.astype(np.float32)
    T = ngf.smooth_random_volume(gi, seed=seed + 1).values.astype(np.float32)
    y = ngf.smooth_random_field(gd, seed=seed + 2, amplitude_mm=2.0).field.astype(np.float32).ravel()
    obj = ngf.LevelObjective.from_device(torch.from_numpy(T).cuda(), torch.from_numpy(R).cuda(),
                                         ngf.build_gather_plan(gd, gi), ngf.NgfParams(), 1.0)
    return obj, y


def _pinned(a):
    t = torch.empty(a.size, dtype=torch.float32, pin_memory=True)
    t.numpy()[:] = a
    return t


@pytest.mark.parametrize("dims,ratio", CASES)
def test_pipeline_bit_identical(dims, ratio):
    obj, y = _setup(dims, ratio)
    h = obj.level.handle
    yp = _pinned(y)
    # the device-resident evaluation on the same y
    x = torch.from_numpy(y).cuda()
    g_dev = torch.empty_like(x)
    sc = torch.zeros(3, dtype=torch.float64, device="cuda")
    obj.eval_device(x, g_dev, sc)
    J_dev, g_dev = float(sc[0].item()), g_dev.cpu().numpy()
    for parts in (1, 2, 3, 4, 5, 8):
        assert lib().ngf_level_set_host_pipeline(h, parts) == 0
        for _ in range(2):  # the second call reuses the streams / events
            J, g = obj(yp.numpy())
            assert J == J_dev, (parts, J, J_dev)
            assert np.array_equal(g, g_dev), (parts, float(np.abs(g - g_dev).max()))
    # a pageable y runs the serial path: same numbers
    assert lib().ngf_level_set_host_pipeline(h, 3) == 0
    J, g = obj(y.copy())
    assert J == J_dev and np.array_equal(g, g_dev)


def test_pipeline_nonfinite_trial_point():
    obj, y = _setup((128, 128, 128), 4)
    h = obj.level.handle
    n = y.size // 3
    for where in (5, n - 7, 2 * n + n // 2):  # first, last part; z component
        yb = y.copy()
        yb[where] = np.nan
        for parts in (1, 3):
            assert lib().ngf_level_set_host_pipeline(h, parts) == 0
            J, g = obj(_pinned(yb).numpy())
            assert J == float("inf") and not g.any()
        # the flag is re-armed: a finite point after it evaluates normally
        J, _ = obj(_pinned(y).numpy())
        assert np.isfinite(J)


def test_pipeline_argument_checks():
    obj, _ = _setup((64, 64, 64), 4)
    assert lib().ngf_level_set_host_pipeline(obj.level.handle, -1) < 0
    assert lib().ngf_level_set_host_pipeline(obj.level.handle, 9) < 0
    assert lib().ngf_level_set_host_pipeline(None, 2) < 0
