"""Pin the CPU oracle against the real reference (CPU only, no GPU).

Every comparison is bit-exact (np.array_equal / float ==): the oracle is a
restatement of the reference arithmetic, so any difference is an oracle bug.
Fixtures come from tests/golden/make_golden.py, which ran /root/reference.
"""

import numpy as np
import pytest

from conftest import grid_from, load_golden
from oracle import ngf_oracle as O

PRECS = ("f32", "f64")


def test_reference_recorded_checksums():
    """The reference's own recorded benchmark checksums
    (/root/reference/pkg/test_output.txt:29-40, f64, 32^3, seed 0)."""
    g = O.grid((32, 32, 32))
    gd = O.def_grid_for(g, 4)
    R = O.smooth_random_volume(g, 0)
    T = O.smooth_random_volume(g, 1)
    y = O.smooth_random_field(gd, 2, 2.0)
    yhat = O.apply_P(y, gd, g)
    assert O.checksum(yhat) == "e5b27dd91b2bf292"
    assert O.checksum(O.apply_Pt(yhat, gd, g)) == "44048d52daeb722a"
    gR, nR = O.ref_terms(R, g, 10.0)
    _, grad = O.distance_and_gradient(y, gd, T, g, gR, nR)
    assert O.checksum(grad) == "d92bcb33030e610b"
    yy, _, _ = O.register(R, T, g, lbfgs_cfg=dict(max_iterations=3))
    assert O.checksum(yy) == "e70268ad7b5c9f9a"


def test_transfer_golden():
    z = load_golden("transfer")
    for k in range(int(z["n"])):
        gd, gi = grid_from(z[f"{k}_gd"]), grid_from(z[f"{k}_gi"])
        plan = O.gather_plan(gd, gi)
        for a in range(3):
            i0, w1 = O.axis_transfer(gi, gd, a)
            assert np.array_equal(i0, z[f"{k}_i0_{a}"])
            assert np.array_equal(w1, z[f"{k}_w1_{a}"])
            st, cnt, w = plan[a]
            assert np.array_equal(st, z[f"{k}_start_{a}"])
            assert np.array_equal(cnt, z[f"{k}_counts_{a}"])
            assert np.array_equal(w, z[f"{k}_weights_{a}"])
        for p in PRECS:
            assert np.array_equal(O.apply_P(z[f"{k}_y_{p}"], gd, gi), z[f"{k}_P_{p}"])
            assert np.array_equal(O.apply_Pt(z[f"{k}_r_{p}"], gd, gi, plan), z[f"{k}_Pt_{p}"])
            # scatter / red-black variants (transfer.py:199-256), one worker
            assert np.array_equal(O.apply_Pt_scatter(z[f"{k}_r_{p}"], gd, gi), z[f"{k}_Pts_{p}"])
            assert np.array_equal(O.apply_Pt_redblack(z[f"{k}_r_{p}"], gd, gi), z[f"{k}_Ptrb_{p}"])


def test_warp_golden():
    z = load_golden("warp")
    for k in range(int(z["n"])):
        g = grid_from(z[f"{k}_g"])
        for p in PRECS:
            T, yh, s = z[f"{k}_T_{p}"], z[f"{k}_yhat_{p}"], z[f"{k}_s_{p}"]
            W, mask = O.warp(T, g, yh)
            assert np.array_equal(W, z[f"{k}_W_{p}"])
            assert np.array_equal(mask, z[f"{k}_mask_{p}"])
            assert np.array_equal(O.warp_jt(T, g, yh, s), z[f"{k}_Jt_{p}"])
            assert np.array_equal(O.gradient(T, g.spacing), z[f"{k}_G_{p}"])
            assert np.array_equal(O.gradient_t(z[f"{k}_q_{p}"], g.spacing), z[f"{k}_Gt_{p}"])


def test_warp_workers_bit_identical():
    z = load_golden("warp")
    g = grid_from(z["0_g"])
    W1, _ = O.warp(z["0_T_f32"], g, z["0_yhat_f32"], workers=1)
    W4, _ = O.warp(z["0_T_f32"], g, z["0_yhat_f32"], workers=4)
    assert np.array_equal(W1, W4)


def test_ngf_golden():
    z = load_golden("ngf")
    for k in range(int(z["n"])):
        gi, gd = grid_from(z[f"{k}_gi"]), grid_from(z[f"{k}_gd"])
        for p in PRECS:
            R, T, y = z[f"{k}_R_{p}"], z[f"{k}_T_{p}"], z[f"{k}_y_{p}"]
            gR, nR = O.ref_terms(R, gi, 10.0)
            assert np.array_equal(gR, z[f"{k}_gR_{p}"])
            assert np.array_equal(nR, z[f"{k}_nR_{p}"])
            D, gD = O.distance_and_gradient(y, gd, T, gi, gR, nR)
            assert D == float(z[f"{k}_D_{p}"])
            assert np.array_equal(gD, z[f"{k}_gD_{p}"])
            obj = O.Objective(T, R, gd, gi)
            J, gJ = obj(y.ravel())
            assert J == float(z[f"{k}_J_{p}"])
            assert obj.last_D == float(z[f"{k}_Jd_{p}"])
            assert obj.last_S == float(z[f"{k}_Js_{p}"])
            assert np.array_equal(gJ, z[f"{k}_gJ_{p}"])


def test_ngf_orthogonal_ramps_closed_form():
    z = load_golden("ngf")
    g = O.grid((6, 6, 6))
    x = O.centers(g, 0)[None, None, :] + np.zeros(O.shape_of(g))
    y = O.centers(g, 1)[None, :, None] + np.zeros(O.shape_of(g))
    gR, nR = O.ref_terms(y, g, 0.1)
    W, _ = O.warp(x, g, O.identity(g))
    D = O.ngf_value(W, g, gR, nR, 0.1, 0.1)
    assert D == float(z["ramp_D"])
    expected = 0.5 * (1.0 - (0.01 / 1.01) ** 2) * 216
    assert abs(D - expected) < 1e-10 * expected


def test_curvature_golden():
    z = load_golden("curvature")
    for k in range(int(z["n"])):
        g = grid_from(z[f"{k}_g"])
        for p in PRECS:
            y = z[f"{k}_y_{p}"]
            assert O.curvature_value(y, g) == float(z[f"{k}_S_{p}"])
            assert np.array_equal(O.curvature_gradient(y, g), z[f"{k}_gS_{p}"])
            u = (y - O.identity(g, y.dtype))[0]
            assert np.array_equal(O.laplacian(u, g), z[f"{k}_L_{p}"])
            assert np.array_equal(O.laplacian_t(u, g), z[f"{k}_LT_{p}"])


def test_multilevel_golden():
    z = load_golden("multilevel")
    g = O.grid((7, 8, 5), (1.0, 1.2, 2.0), (0.3, -1.0, 2.5))
    for p in PRECS:
        pyr = O.pyramid(z[f"pyr_in_{p}"], g, 3)
        for k, (v, gg) in enumerate(pyr):
            assert np.array_equal(v, z[f"pyr_{k}_{p}"])
            assert np.array_equal(np.array([*gg.dims, *gg.spacing, *gg.origin]), z[f"pyr_{k}_g"])
        v, gg = O.downsample(z[f"ds_in_{p}"], grid_from(z["ds_g_in"]))
        assert np.array_equal(v, z[f"ds_out_{p}"])
        assert np.array_equal(np.array([*gg.dims, *gg.spacing, *gg.origin]), z["ds_g_out"])
    for dims, lv in zip(z["auto_dims"], z["auto_levels"]):
        assert O.auto_levels(tuple(int(d) for d in dims), 16) == int(lv)
    for k in range(4):
        gi = grid_from(z[f"defgrid_{k}_gi"])
        for ratio in (2, 4, 8):
            gd = O.def_grid_for(gi, ratio)
            assert np.array_equal(np.array([*gd.dims, *gd.spacing, *gd.origin]),
                                  z[f"defgrid_{k}_{ratio}"])
    gc, gf = grid_from(z["pro_gc"]), grid_from(z["pro_gf"])
    for p in PRECS:
        assert np.array_equal(O.prolong(z[f"pro_in_{p}"], gc, gf), z[f"pro_out_{p}"])


def test_lbfgs_golden():
    z = load_golden("lbfgs")
    for p in PRECS:
        hist = [(z[f"tl_s{k}_{p}"], z[f"tl_y{k}_{p}"]) for k in range(5)]
        assert np.array_equal(O.two_loop(hist, z[f"tl_g_{p}"]), z[f"tl_d_{p}"])
    A, b = z["quad_A"], z["quad_b"]

    def f(x):
        return 0.5 * float(x @ (A @ x)) - float(b @ x), A @ x - b

    x, recs, reason, failed = O.lbfgs(f, np.zeros(12))
    assert np.array_equal(x, z["quad_x"])
    assert np.array_equal(np.array(recs, dtype=float), z["quad_recs"])
    assert reason == str(z["quad_reason"])
    assert not failed


@pytest.mark.slow
def test_register_golden():
    z = load_golden("register")
    g = grid_from(z["g"])
    for p in PRECS:
        y, gd, info = O.register(z["R"], z["T"], g, coarsest_min_dim=8, precision=p,
                                 lbfgs_cfg=dict(max_iterations=30))
        assert np.array_equal(y, z[f"y_{p}"])
        assert [lv["iterations"] for lv in info] == list(z[f"iters_{p}"])
        assert [lv["stop_reason"] for lv in info] == list(z[f"reasons_{p}"])
        assert [lv["records"][-1][1] for lv in info] == list(z[f"J_{p}"])


def test_dense_P_matches_apply():
    rng = np.random.default_rng(5)
    z = load_golden("transfer")
    for k in range(12):
        gd, gi = grid_from(z[f"{k}_gd"]), grid_from(z[f"{k}_gi"])
        if np.prod(gi.dims) > 512:
            continue
        P = O.dense_P(gd, gi)
        r = rng.standard_normal((3,) + O.shape_of(gi))
        out = O.apply_Pt(r, gd, gi)
        for c in range(3):
            ref = (P.T @ r[c].ravel()).reshape(O.shape_of(gd))
            assert np.max(np.abs(out[c] - ref)) < 1e-13 * (np.abs(ref).max() + 1)
