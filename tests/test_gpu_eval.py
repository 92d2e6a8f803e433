"""Level objective (objective.py:22-60) on the device: the fused performance path
within the north-star tolerances (J 1e-4 relative, grad 1e-3 relative L2 vs the
f32 oracle), the exact path bit-identical to the reference, determinism, the
non-finite guard and the edge shapes the reference tests exercise."""

import numpy as np
import pytest
import torch

from conftest import load_golden

pytestmark = pytest.mark.gpu

import paper_1812_06765_b200 as ngf  # noqa: E402
from oracle import ngf_oracle as O  # noqa: E402

TOL_J = 1e-4      # north star: objective within 1e-4 relative (fp32 vs reference)
TOL_G = 1e-3      # north star: gradient within 1e-3 relative L2


def _g(arr):
    a = np.asarray(arr, dtype=np.float64)
    return ngf.Grid3(tuple(int(v) for v in a[:3]), tuple(a[3:6]), tuple(a[6:9]))


def _og(g):
    return O.grid(g.dims, g.spacing, g.origin)


def _device_obj(T, R, gd, gi, exact=False, alpha=1.0, params=ngf.NgfParams()):
    plan = ngf.build_gather_plan(gd, gi)
    return ngf.LevelObjective.from_device(torch.from_numpy(np.ascontiguousarray(T)).cuda(),
                                          torch.from_numpy(np.ascontiguousarray(R)).cuda(),
                                          plan, params, alpha, exact=exact)


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


@pytest.mark.parametrize("k", [0, 1, 2, 3])
@pytest.mark.parametrize("p", ["f32", "f64"])
def test_objective_golden(k, p):
    """Fixtures from the reference's LevelObjective: fused within tolerance, exact bit-equal."""
    z = load_golden("ngf")
    gi, gd = _g(z[f"{k}_gi"]), _g(z[f"{k}_gd"])
    R, T, y = z[f"{k}_R_{p}"], z[f"{k}_T_{p}"], z[f"{k}_y_{p}"]
    J_ref, g_ref = float(z[f"{k}_J_{p}"]), z[f"{k}_gJ_{p}"]
    fused = _device_obj(T, R, gd, gi)
    J, g = fused(y.ravel())
    assert abs(J - J_ref) <= TOL_J * abs(J_ref)
    assert _rel(g, g_ref) <= TOL_G
    if p == "f64":  # f64 fused is far tighter than the f32 bar
        assert abs(J - J_ref) <= 1e-10 * abs(J_ref) and _rel(g, g_ref) <= 1e-10
    exact = _device_obj(T, R, gd, gi, exact=True)
    Je, ge = exact(y.ravel())
    assert Je == J_ref
    assert np.array_equal(ge, g_ref)
    assert exact.last_D == float(z[f"{k}_Jd_{p}"]) and exact.last_S == float(z[f"{k}_Js_{p}"])
    # the exact path with the red-black P^T equals the reference's red-black objective
    plan = ngf.build_gather_plan(gd, gi)
    rb = ngf.LevelObjective.from_device(torch.from_numpy(np.ascontiguousarray(T)).cuda(),
                                        torch.from_numpy(np.ascontiguousarray(R)).cuda(), plan,
                                        ngf.NgfParams(), 1.0, exact=True, pt_variant="redblack")
    Jrb, grb = rb(y.ravel())
    assert Jrb == float(z[f"{k}_Jrb_{p}"])
    assert np.array_equal(grb, z[f"{k}_gJrb_{p}"])


def test_objective_from_reference_terms_matches_from_R():
    """LevelObjective built like the reference (template, ReferenceTerms, plan) equals
    the device-resident constructor."""
    z = load_golden("ngf")
    gi, gd = _g(z["0_gi"]), _g(z["0_gd"])
    R, T, y = z["0_R_f32"], z["0_T_f32"], z["0_y_f32"]
    params = ngf.NgfParams()
    ref = ngf.precompute_reference_terms(ngf.Image3(gi, R), params)
    obj = ngf.LevelObjective(template=ngf.Image3(gi, T), ref=ref,
                             plan=ngf.build_gather_plan(gd, gi), params=params, alpha=1.0)
    J1, g1 = obj(y.ravel())
    J2, g2 = _device_obj(T, R, gd, gi)(y.ravel())
    assert J1 == J2 and np.array_equal(g1, g2)


@pytest.mark.parametrize("dims,ratio,dd", [
    ((64, 64, 64), 4, None),        # C1 shape
    ((70, 45, 33), 4, None),        # ragged, several partial tiles
    ((40, 40, 40), 1, None),        # def grid == image grid (ratio 1)
    ((50, 30, 20), 3, None),        # non power-of-two ratio
    ((48, 40, 36), 2, None),        # ratio 2 (config 2: 64^3 def grid on 128^3)
    ((33, 33, 33), None, (17, 17, 17)),  # 65^3-on-128^3 style (width-5 gather)
    ((24, 20, 1), 4, None),         # degenerate z
    ((48, 36, 28), 16, None),       # very coarse def grid (wide windows)
])
def test_fused_vs_oracle_shapes(dims, ratio, dd):
    gi = ngf.Grid3(dims, (1.0, 1.1, 0.9), (-3.0, 2.0, 1.0))
    if ratio:
        gd = ngf.deformation_grid_for(gi, ratio)
    else:
        hd = tuple(n * s / m for n, s, m in zip(gi.dims, gi.spacing, dd))
        od = tuple(o - s / 2 + sd / 2 for o, s, sd in zip(gi.origin, gi.spacing, hd))
        gd = ngf.Grid3(dd, hd, od)
    R = ngf.smooth_random_volume(gi, seed=5).values.astype(np.float32)
    T = ngf.smooth_random_volume(gi, seed=6).values.astype(np.float32)
    y = ngf.smooth_random_field(gd, seed=7, amplitude_mm=2.5).field.astype(np.float32)
    J_ref, g_ref = O.Objective(T, R, _og(gd), _og(gi))(y.ravel())
    J, g = _device_obj(T, R, gd, gi)(y.ravel())
    assert abs(J - J_ref) <= TOL_J * abs(J_ref), (J, J_ref)
    assert _rel(g, g_ref) <= TOL_G
    Je, ge = _device_obj(T, R, gd, gi, exact=True)(y.ravel())
    assert Je == J_ref and np.array_equal(ge, g_ref)


def test_fused_is_deterministic():
    gi = ngf.Grid3((64, 64, 64), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    gd = ngf.deformation_grid_for(gi, 4)
    R = ngf.smooth_random_volume(gi, seed=1).values.astype(np.float32)
    T = ngf.smooth_random_volume(gi, seed=2).values.astype(np.float32)
    y = ngf.smooth_random_field(gd, seed=3, amplitude_mm=2.0).field.astype(np.float32)
    obj = _device_obj(T, R, gd, gi)
    J1, g1 = obj(y.ravel())
    for _ in range(3):
        J2, g2 = obj(y.ravel())
        assert J1 == J2 and np.array_equal(g1, g2)


def test_non_finite_trial_point_forces_backtrack():
    gi = ngf.Grid3((16, 16, 16), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    gd = ngf.deformation_grid_for(gi, 4)
    T = ngf.smooth_random_volume(gi, seed=1).values.astype(np.float32)
    obj = _device_obj(T, T, gd, gi)
    y = ngf.make_identity(gd, np.float32).field.ravel().copy()
    y[5] = np.inf
    J, g = obj(y)
    assert J == float("inf") and not np.any(g)
    # device path: J = inf comes back from the kernel itself
    x = torch.from_numpy(y).cuda()
    gd_ = torch.empty_like(x)
    sc = obj.eval_device(x, gd_).cpu().numpy()
    assert sc[0] == np.inf
    y[5] = 0.5
    J2, _ = obj(y)
    assert np.isfinite(J2)  # flag was reset


def test_matched_images_identity_is_stationary():
    # tests/test_ngf.py:80-87: T == R, tau == rho, identity -> zero gradient
    g = ngf.Grid3((24, 24, 24), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    T = ngf.smooth_random_volume(g, seed=22).values
    params = ngf.NgfParams(5.0, 5.0)
    obj = _device_obj(T, T, g, g, params=params)
    J, grad = obj(ngf.make_identity(g).field.ravel())
    assert abs(J) < 1e-10 and np.max(np.abs(grad)) < 1e-12
    obj = _device_obj(T, T, g, g, params=params, exact=True)
    J, grad = obj(ngf.make_identity(g).field.ravel())
    assert abs(J) < 1e-12 and np.max(np.abs(grad)) < 1e-12


def test_gradient_matches_finite_differences_f64():
    # tests/test_acceptance.py:176-237 style: fused f64 gradient vs central differences of J
    gi = ngf.Grid3((10, 9, 8), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    gd = ngf.Grid3((4, 3, 3), tuple(n / m for n, m in zip(gi.dims, (4, 3, 3))),
                   tuple(-0.5 + n / m / 2 for n, m in zip(gi.dims, (4, 3, 3))))
    T = ngf.smooth_random_volume(gi, seed=11).values
    R = ngf.smooth_random_volume(gi, seed=12).values
    rng = np.random.default_rng(303)
    ident = ngf.identity_field_array(gd)
    center = np.array([o + e / 2 for o, e in zip(gi.origin, gi.extent)])
    field = center[:, None, None, None] + 0.78 * (ident - center[:, None, None, None])
    field = field + rng.uniform(-0.12, 0.12, field.shape)
    obj = _device_obj(T, R, gd, gi)
    x0 = field.ravel()
    _, grad = obj(x0)
    eps = 1e-6
    fd = np.empty_like(grad)
    for i in range(x0.size):
        xp = x0.copy()
        xp[i] += eps
        xm = x0.copy()
        xm[i] -= eps
        fd[i] = (obj(xp)[0] - obj(xm)[0]) / (2 * eps)
    assert np.abs(fd - grad).max() / np.abs(grad).max() < 1e-6


@pytest.mark.parametrize("dims,spacing,ratio", [((70, 50, 37), (1.0, 1.0, 1.0), 4),
                                                ((64, 40, 33), (0.75, 1.1, 1.3), 3),
                                                ((48, 1, 40), (1.0, 1.0, 1.0), 4),
                                                ((33, 29, 30), (1.0, 1.0, 1.0), 1)])
def test_packed_march_matches_scalar_march(monkeypatch, dims, spacing, ratio):
    """The opt-in two-slot float2 march (FFMA2/FADD2/FMUL2): the forward terms are
    bit-identical to the scalar march, the gradient agrees to f32 rounding (incl.
    non-power-of-two spacing and a degenerate axis)."""
    gi = ngf.Grid3(dims, spacing, (0.5, -1.0, 2.0))
    gd = ngf.deformation_grid_for(gi, ratio)
    R = ngf.smooth_random_volume(gi, seed=7).values.astype(np.float32)
    T = ngf.smooth_random_volume(gi, seed=8).values.astype(np.float32)
    y = ngf.smooth_random_field(gd, seed=9, amplitude_mm=2.0).field.astype(np.float32)
    x = torch.from_numpy(y.ravel().copy()).cuda()
    monkeypatch.setenv("NGF_FUSED_VARIANT", "1")  # the shape the packed march is built for
    out = []
    for packed in (False, True):
        if packed:
            monkeypatch.setenv("NGF_FUSED_PACKED", "1")
        else:
            monkeypatch.delenv("NGF_FUSED_PACKED", raising=False)
        obj = _device_obj(T, R, gd, gi)
        g = torch.empty_like(x)
        sc = obj.eval_device(x, g).cpu().numpy().copy()
        out.append((sc, g.cpu().numpy()))
    assert out[0][0][1] == out[1][0][1]  # D: forward terms bit-identical
    assert np.max(np.abs(out[0][1] - out[1][1])) <= 1e-5 * np.max(np.abs(out[0][1]))


@pytest.mark.parametrize("variant,prec", [("0", "f32"), ("1", "f32"), ("2", "f32"), ("3", "f32"),
                                          ("4", "f32"), ("5", "f32"),
                                          ("0", "f64"), ("4", "f64"), ("5", "f64")])
@pytest.mark.parametrize("dims,ratio", [((40, 40, 40), 1), ((70, 45, 33), 4)])
def test_every_kernel_variant_within_tolerance(monkeypatch, variant, prec, dims, ratio):
    """Each tile/occupancy variant of the fused march (forced with NGF_FUSED_VARIANT),
    incl. ratio 1 on non-unit spacing where the index map can advance by 2 (widest windows)."""
    monkeypatch.setenv("NGF_FUSED_VARIANT", variant)
    gi = ngf.Grid3(dims, (1.0, 1.1, 0.9), (-3.0, 2.0, 1.0))
    gd = ngf.deformation_grid_for(gi, ratio)
    dt = np.float32 if prec == "f32" else np.float64
    R = ngf.smooth_random_volume(gi, seed=5).values.astype(dt)
    T = ngf.smooth_random_volume(gi, seed=6).values.astype(dt)
    y = ngf.smooth_random_field(gd, seed=7, amplitude_mm=2.5).field.astype(dt)
    J_ref, g_ref = O.Objective(T, R, _og(gd), _og(gi))(y.ravel())
    J, g = _device_obj(T, R, gd, gi)(y.ravel())
    tol_J, tol_G = (TOL_J, TOL_G) if prec == "f32" else (1e-10, 1e-10)
    assert abs(J - J_ref) <= tol_J * abs(J_ref), (J, J_ref)
    assert _rel(g, g_ref) <= tol_G
