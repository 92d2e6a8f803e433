"""L-BFGS driver edge cases against the reference's lbfgs_minimize (lbfgs.py:94-181):
a zero line-search budget evaluates no trial point and reports a failed line search,
in the Python loop, the native loop and the graph loop alike."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_1812_06765_b200 as ngf  # noqa: E402
from paper_1812_06765_b200._lib import lib  # noqa: E402
from oracle import ref as oref  # noqa: E402


def _quadratic(n=50, seed=3):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((n, n))
    H = A @ A.T / n + np.eye(n)
    b = rng.standard_normal(n)
    return (lambda x: (float(0.5 * x @ H @ x - b @ x), H @ x - b)), rng.standard_normal(n)


@pytest.mark.parametrize("ls", [0, -1])
def test_zero_line_search_budget_python_loop(ls):
    f, x0 = _quadratic()
    x, tr = ngf.lbfgs_minimize(f, x0, ngf.LbfgsConfig(max_ls_steps=ls))
    assert tr.stop_reason == "line search failed" and tr.line_search_failed
    assert len(tr.records) == 0 and np.array_equal(x, x0)
    rm = oref.load()
    if rm is not None:
        from ngfreg import lbfgs as rl
        xr, trr = rl.lbfgs_minimize(f, x0, rl.LbfgsConfig(max_ls_steps=ls))
        assert trr.stop_reason == tr.stop_reason and len(trr.records) == 0 and np.array_equal(xr, x)


@pytest.mark.parametrize("graph", [0, 1])
def test_zero_line_search_budget_native_loop(graph):
    gi = ngf.Grid3((24, 24, 24), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    gd = ngf.deformation_grid_for(gi, 4)
    R = ngf.smooth_random_volume(gi, seed=1).values.astype(np.float32)
    T = ngf.smooth_random_volume(gi, seed=2).values.astype(np.float32)
    obj = ngf.LevelObjective.from_device(torch.from_numpy(T).cuda(), torch.from_numpy(R).cuda(),
                                         ngf.build_gather_plan(gd, gi), ngf.NgfParams(), 1.0)
    y0 = ngf.identity_field_array(gd, np.float32).ravel()
    prev = lib().ngf_lbfgs_set_graph(graph)
    try:
        x, tr = ngf.lbfgs_minimize(obj, y0, ngf.LbfgsConfig(max_ls_steps=0))
    finally:
        lib().ngf_lbfgs_set_graph(prev)
    assert tr.stop_reason == "line search failed" and tr.line_search_failed
    assert len(tr.records) == 0 and tr.evaluations == 1 and np.array_equal(x, y0)
