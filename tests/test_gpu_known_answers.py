"""The reference's own known-answer tests, run on the device path.

Each test restates one of the reference's analytic checks against the sm_100a kernels
(numpy in -> device -> numpy out): closed-form NGF on orthogonal ramps
(tests/test_ngf.py:35-46), P / P^T adjointness on random grid pairs
(tests/test_transfer.py:127-136), trilinear exactness of the warp
(tests/test_warp.py:25-39), the warp Jacobian^T against finite differences
(tests/test_warp.py:64-88) and the curvature null space of affine maps
(tests/test_curvature.py:23-32).  The same closed forms are also checked through the
fused LevelObjective, which shares none of the standalone operator kernels.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_1812_06765_b200 as ngf  # noqa: E402


def _grid(dims, spacing=(1.0, 1.0, 1.0), origin=(0.0, 0.0, 0.0)):
    return ngf.Grid3(tuple(dims), tuple(spacing), tuple(origin))


def _ramps(g, dtype):
    x = g.axis_centers(0)[None, None, :]
    y = g.axis_centers(1)[None, :, None]
    T = (x + np.zeros(g.shape)).astype(dtype)
    R = (y + np.zeros(g.shape)).astype(dtype)
    return T, R


def _random_grid_pair(rng, max_dim=9):
    """(def_grid, image_grid) covering the same world box (reference tests/conftest.py:12-21)."""
    di = tuple(int(v) for v in rng.integers(1, max_dim + 1, 3))
    dd = tuple(int(rng.integers(1, v + 1)) for v in di)
    h = tuple(float(v) for v in rng.uniform(0.5, 3.0, 3))
    o = tuple(float(v) for v in rng.uniform(-5, 5, 3))
    hd = tuple(n * s / m for n, s, m in zip(di, h, dd))
    od = tuple(oo - s / 2 + sd / 2 for oo, s, sd in zip(o, h, hd))
    return _grid(dd, hd, od), _grid(di, h, o)


def test_orthogonal_ramps_closed_form_exact_path():
    """T = x, R = y, tau = rho = 0.1: every voxel contributes 1 - (0.01/1.01)^2."""
    g = _grid((6, 6, 6))
    T, R = _ramps(g, np.float64)
    params = ngf.NgfParams(0.1, 0.1)
    ref = ngf.precompute_reference_terms(ngf.Image3(g, R), params)
    warped = ngf.warp_image(ngf.Image3(g, T), ngf.make_identity(g))
    h_bar = g.cell_volume
    expected = h_bar / 2 * (1.0 - (0.01 / 1.01) ** 2) * g.num_points
    assert abs(ngf.ngf_value(warped, ref, params, h_bar) - expected) < 1e-10 * expected


@pytest.mark.parametrize("dtype,tol", [(np.float64, 1e-10), (np.float32, 1e-5)])
def test_orthogonal_ramps_closed_form_fused(dtype, tol):
    """Same closed form through the fused evaluation (identity y on a grid-ratio-1
    deformation grid, alpha = 0, so J = D)."""
    g = _grid((12, 10, 9))
    T, R = _ramps(g, dtype)
    params = ngf.NgfParams(0.1, 0.1)
    plan = ngf.build_gather_plan(g, g)
    obj = ngf.LevelObjective.from_device(torch.from_numpy(T).cuda(), torch.from_numpy(R).cuda(),
                                         plan, params, 0.0)
    J, grad = obj(ngf.make_identity(g).field.astype(dtype).ravel())
    expected = g.cell_volume / 2 * (1.0 - (0.01 / 1.01) ** 2) * g.num_points
    assert abs(J - expected) < tol * expected
    assert np.all(np.isfinite(grad))


def test_adjoint_identity_on_device():
    """<P y, z> == <y, P^T z> for every P^T variant, f64, 20 random grid pairs."""
    rng = np.random.default_rng(7)
    for _ in range(20):
        gd, gi = _random_grid_pair(rng)
        plan = ngf.build_gather_plan(gd, gi)
        y = ngf.DeformationField(gd, ngf.make_identity(gd).field + rng.standard_normal((3,) + gd.shape))
        z = ngf.VectorField3(gi, rng.standard_normal((3,) + gi.shape))
        lhs = float(np.sum(ngf.apply_P(y, gi).field * z.field))
        for out in (ngf.apply_Pt_gather(z, plan), ngf.apply_Pt(z, plan, "redblack"),
                    ngf.apply_Pt(z, plan, "scatter")):
            rhs = float(np.sum(y.field * out.field))
            assert abs(lhs - rhs) <= 1e-12 * (abs(lhs) + 1), (gd.dims, gi.dims)


def test_warp_exact_on_trilinear_images():
    """The interpolant reproduces functions linear per axis exactly (f64, 1e-10)."""
    rng = np.random.default_rng(3)
    g = _grid((7, 6, 5), (1.0, 1.2, 0.9), (0.0, -1.0, 2.0))
    x = g.axis_centers(0)[None, None, :]
    y = g.axis_centers(1)[None, :, None]
    z = g.axis_centers(2)[:, None, None]
    vals = 2.0 * x - 3.0 * y + 0.5 * z + 0.25 * x * y + 1.0
    T = ngf.Image3(g, vals + np.zeros(g.shape))
    field = ngf.make_identity(g).field + rng.uniform(-0.3, 0.3, (3,) + g.shape)
    res = ngf.warp_image(T, ngf.DeformationField(g, field))
    expected = 2.0 * field[0] - 3.0 * field[1] + 0.5 * field[2] + 0.25 * field[0] * field[1] + 1.0
    inside = res.inside_mask
    assert inside.sum() > g.num_points // 2
    assert np.allclose(res.warped.values[inside], expected[inside], atol=1e-10)
    assert np.all(res.warped.values[~inside] == 0.0)


def test_warp_jacobian_transpose_matches_fd():
    """FD of sum(w * warp(y)) vs the device J^T, away from cell centres and the hull."""
    rng = np.random.default_rng(11)
    g = _grid((8, 7, 6))
    T = ngf.smooth_random_volume(g, seed=11)
    field = ngf.make_identity(g).field + rng.uniform(0.2, 0.4, (3,) + g.shape)
    field = np.clip(field, 0.3, None)
    for a in range(3):
        field[a] = np.minimum(field[a], (g.dims[a] - 1) * g.spacing[a] - 0.3)
    w = rng.standard_normal(g.shape)
    grad = ngf.warp_jacobian_apply_transpose(T, ngf.DeformationField(g, field), w).field
    eps = 1e-6
    for (k, j, i) in [(0, 0, 0), (3, 2, 4), (5, 6, 1)]:
        for a in range(3):
            fp, fm = field.copy(), field.copy()
            fp[a, k, j, i] += eps
            fm[a, k, j, i] -= eps
            vp = ngf.warp_image(T, ngf.DeformationField(g, fp)).warped.values
            vm = ngf.warp_image(T, ngf.DeformationField(g, fm)).warped.values
            fd = np.sum(w * (vp - vm)) / (2 * eps)
            assert abs(fd - grad[a, k, j, i]) < 1e-5 * (abs(fd) + 1), (a, k, j, i)


def test_affine_fields_have_zero_curvature():
    """Linear extrapolation at the boundary keeps affine maps in the null space of L."""
    g = _grid((7, 6, 5), (1.0, 0.9, 1.4))
    A = np.array([[1.1, 0.2, 0.0], [0.0, 0.95, -0.1], [0.05, 0.0, 1.0]])
    b = np.array([2.0, -1.0, 0.5])
    field = np.einsum("cd,dkji->ckji", A, ngf.make_identity(g).field) + b[:, None, None, None]
    y = ngf.DeformationField(g, field)
    assert ngf.curvature_value(y) < 1e-22
    assert np.max(np.abs(ngf.curvature_gradient(y))) < 1e-12
    assert ngf.curvature_value(ngf.make_identity(g)) == 0.0
    assert np.all(ngf.curvature_gradient(ngf.make_identity(g)) == 0)
