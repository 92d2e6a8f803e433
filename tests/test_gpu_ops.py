"""Standalone sm_100a operators vs the reference fixtures: bit-exact (np.array_equal).

Each operator kernel restates the reference's IEEE operation order, so the
device output must equal the reference output byte for byte in f32 and f64,
including the reference's own recorded checksums (pkg/test_output.txt:29-40).
"""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

import paper_1812_06765_b200 as ngf  # noqa: E402
from oracle import ngf_oracle as O  # noqa: E402

PRECS = ("f32", "f64")


def _g(arr):
    a = np.asarray(arr, dtype=np.float64)
    return ngf.Grid3(tuple(int(v) for v in a[:3]), tuple(a[3:6]), tuple(a[6:9]))


def test_reference_checksums_on_device():
    """apply_P, P^T gather and distance_and_gradient reproduce the reference's recorded
    checksums bit for bit (f64, 32^3, seed 0; pkg/test_output.txt:29-33)."""
    g = ngf.Grid3((32, 32, 32), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    gd = ngf.deformation_grid_for(g, 4)
    R = ngf.smooth_random_volume(g, seed=0)
    T = ngf.smooth_random_volume(g, seed=1)
    y = ngf.smooth_random_field(gd, seed=2, amplitude_mm=2.0)
    plan = ngf.build_gather_plan(gd, g)
    yhat = ngf.apply_P(y, g)
    assert O.checksum(yhat.field) == "e5b27dd91b2bf292"
    assert O.checksum(ngf.apply_Pt_gather(yhat, plan).field) == "44048d52daeb722a"
    params = ngf.NgfParams(10.0, 10.0)
    ref = ngf.precompute_reference_terms(R, params)
    _, grad = ngf.distance_and_gradient(y, ref, T, plan, params)
    assert O.checksum(grad.field) == "d92bcb33030e610b"


def test_transfer_bit_exact():
    z = load_golden("transfer")
    for k in range(int(z["n"])):
        gd, gi = _g(z[f"{k}_gd"]), _g(z[f"{k}_gi"])
        plan = ngf.build_gather_plan(gd, gi)
        for p in PRECS:
            y = ngf.DeformationField(gd, z[f"{k}_y_{p}"])
            assert np.array_equal(ngf.apply_P(y, gi).field, z[f"{k}_P_{p}"]), (k, p)
            r = ngf.VectorField3(gi, z[f"{k}_r_{p}"])
            assert np.array_equal(ngf.apply_Pt(r, plan).field, z[f"{k}_Pt_{p}"]), (k, p)
            # red-black: same per-output order as the reference -> bit-identical
            assert np.array_equal(ngf.apply_Pt(r, plan, "redblack").field, z[f"{k}_Ptrb_{p}"]), (k, p)
            assert np.array_equal(ngf.apply_Pt_redblack(r, gd).field, z[f"{k}_Ptrb_{p}"]), (k, p)
            # scatter: float atomics, equal up to reassociation (reference: 1e-12 in f64,
            # benchmark.py:62-85)
            tol = 1e-12 if p == "f64" else 1e-5
            for out in (ngf.apply_Pt(r, plan, "scatter").field, ngf.apply_Pt_scatter_atomic(r, gd).field):
                ref = z[f"{k}_Pts_{p}"].astype(np.float64)
                assert np.max(np.abs(out - ref)) <= tol * (np.abs(ref).max() + 1), (k, p)


def test_warp_and_stencils_bit_exact():
    z = load_golden("warp")
    for k in range(int(z["n"])):
        g = _g(z[f"{k}_g"])
        for p in PRECS:
            T = ngf.Image3(g, z[f"{k}_T_{p}"])
            yh = ngf.VectorField3(g, z[f"{k}_yhat_{p}"])
            res = ngf.warp_image(T, yh)
            assert np.array_equal(res.warped.values, z[f"{k}_W_{p}"]), (k, p)
            assert np.array_equal(res.inside_mask, z[f"{k}_mask_{p}"]), (k, p)
            jt = ngf.warp_jacobian_apply_transpose(T, yh, z[f"{k}_s_{p}"]).field
            assert np.array_equal(jt, z[f"{k}_Jt_{p}"]), (k, p)
            assert np.array_equal(ngf.image_gradient(T).field, z[f"{k}_G_{p}"]), (k, p)
            q = ngf.VectorField3(g, z[f"{k}_q_{p}"])
            assert np.array_equal(ngf.image_gradient_apply_transpose(q, g), z[f"{k}_Gt_{p}"]), (k, p)


def test_ngf_pipeline_bit_exact():
    z = load_golden("ngf")
    for k in range(int(z["n"])):
        gi, gd = _g(z[f"{k}_gi"]), _g(z[f"{k}_gd"])
        for p in PRECS:
            R = ngf.Image3(gi, z[f"{k}_R_{p}"])
            T = ngf.Image3(gi, z[f"{k}_T_{p}"])
            y = ngf.DeformationField(gd, z[f"{k}_y_{p}"])
            params = ngf.NgfParams(10.0, 10.0)
            ref = ngf.precompute_reference_terms(R, params)
            assert np.array_equal(ref.grad.field, z[f"{k}_gR_{p}"])
            assert np.array_equal(ref.norm, z[f"{k}_nR_{p}"])
            plan = ngf.build_gather_plan(gd, gi)
            D, gD = ngf.distance_and_gradient(y, ref, T, plan, params)
            assert D == float(z[f"{k}_D_{p}"]), (k, p)
            assert np.array_equal(gD.field, z[f"{k}_gD_{p}"]), (k, p)


def test_curvature_bit_exact():
    z = load_golden("curvature")
    for k in range(int(z["n"])):
        g = _g(z[f"{k}_g"])
        for p in PRECS:
            y = ngf.DeformationField(g, z[f"{k}_y_{p}"])
            assert ngf.curvature_value(y) == float(z[f"{k}_S_{p}"]), (k, p)
            assert np.array_equal(ngf.curvature_gradient(y), z[f"{k}_gS_{p}"]), (k, p)
            u = (y.field - ngf.identity_field_array(g, y.field.dtype))[0]
            assert np.array_equal(ngf.apply_laplacian(u, g), z[f"{k}_L_{p}"])
            assert np.array_equal(ngf.apply_laplacian_transpose(u, g), z[f"{k}_LT_{p}"])


def test_pyramid_and_prolongation_bit_exact():
    z = load_golden("multilevel")
    g = ngf.Grid3((7, 8, 5), (1.0, 1.2, 2.0), (0.3, -1.0, 2.5))
    for p in PRECS:
        pyr = ngf.build_pyramid(ngf.Image3(g, z[f"pyr_in_{p}"]), 3)
        for k, lv in enumerate(pyr):
            assert np.array_equal(lv.values, z[f"pyr_{k}_{p}"]), (k, p)
        ds = ngf.downsample_image(ngf.Image3(_g(z["ds_g_in"]), z[f"ds_in_{p}"]))
        assert np.array_equal(ds.values, z[f"ds_out_{p}"])
        y = ngf.DeformationField(_g(z["pro_gc"]), z[f"pro_in_{p}"])
        out = ngf.prolong_deformation(y, _g(z["pro_gf"]))
        assert np.array_equal(out.field, z[f"pro_out_{p}"]), p
    # identity prolongs to identity bit-exactly (tests/test_multilevel.py:73-77)
    coarse = ngf.deformation_grid_for(ngf.Grid3((16, 16, 16), (1, 1, 1), (0, 0, 0)), 8)
    fine = ngf.deformation_grid_for(ngf.Grid3((16, 16, 16), (1, 1, 1), (0, 0, 0)), 4)
    out = ngf.prolong_deformation(ngf.make_identity(coarse), fine)
    assert np.array_equal(out.field, ngf.make_identity(fine).field)


def test_two_loop_matches_reference():
    z = load_golden("lbfgs")
    for p in PRECS:
        hist = [(z[f"tl_s{k}_{p}"], z[f"tl_y{k}_{p}"]) for k in range(5)]
        d = ngf.two_loop_direction(hist, z[f"tl_g_{p}"])
        ref = z[f"tl_d_{p}"]
        tol = 1e-5 if p == "f32" else 1e-12
        assert np.max(np.abs(d - ref)) <= tol * np.abs(ref).max(), p
    g = np.random.default_rng(0).standard_normal(8)
    assert np.array_equal(ngf.two_loop_direction([], g), -g)


def test_lbfgs_quadratic_trace_matches_reference():
    z = load_golden("lbfgs")
    A, b = z["quad_A"], z["quad_b"]

    def f(x):
        return 0.5 * float(x @ (A @ x)) - float(b @ x), A @ x - b

    x, trace = ngf.lbfgs_minimize(f, np.zeros(12))
    recs = z["quad_recs"]
    assert trace.iterations == len(recs)
    assert trace.stop_reason == str(z["quad_reason"])
    assert np.max(np.abs(x - z["quad_x"])) < 1e-9
    for r, row in zip(trace.records, recs):
        assert r.ls_evals == int(row[4]) and r.step == row[3]
        assert abs(r.J - row[1]) <= 1e-10 * (abs(row[1]) + 1)


def test_lbfgs_line_search_failure_and_stationary_start():
    def up(x):
        return float(np.sum(x)), -np.ones_like(x)

    x, trace = ngf.lbfgs_minimize(up, np.ones(3), cfg=ngf.LbfgsConfig(max_ls_steps=5))
    assert trace.line_search_failed and trace.stop_reason == "line search failed"
    assert np.array_equal(x, np.ones(3))

    def flat(x):
        return 0.0, np.zeros_like(x)

    x, trace = ngf.lbfgs_minimize(flat, np.ones(4))
    assert trace.iterations == 0 and trace.stop_reason == "stationary start"
