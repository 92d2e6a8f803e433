"""Generate golden fixtures by running the REAL reference package (build container only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Imports `ngfreg` from /root/reference/pkg/src (read-only) and writes small
.npz files next to this script.  The GPU box never runs this; the tests only
read the committed .npz files.  Every case here mirrors a reference test or a
SURVEY.md §8 row; inputs are stored alongside outputs so the oracle and the
CUDA path can be fed identical bytes.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from ngfreg import curvature, lbfgs, multilevel, ngf, synthetic, transfer, warp  # noqa: E402
from ngfreg.geometry import DeformationField, Grid3, Image3, VectorField3, make_identity  # noqa: E402
from ngfreg.objective import LevelObjective  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
DTYPES = {"f32": np.float32, "f64": np.float64}


def garr(g: Grid3):
    return np.array([*g.dims, *g.spacing, *g.origin], dtype=np.float64)


def random_pair(rng, max_dim=9):
    # same construction as the reference's tests/conftest.py:12-21
    di = tuple(int(x) for x in rng.integers(1, max_dim + 1, 3))
    dd = tuple(int(rng.integers(1, v + 1)) for v in di)
    h = tuple(float(x) for x in rng.uniform(0.5, 3.0, 3))
    o = tuple(float(x) for x in rng.uniform(-5, 5, 3))
    gi = Grid3(di, h, o)
    hd = tuple(n * s / m for n, s, m in zip(di, h, dd))
    od = tuple(oo - s / 2 + sd / 2 for oo, s, sd in zip(o, h, hd))
    return Grid3(dd, hd, od), gi


def def_like(gi: Grid3, dd):
    hd = tuple(n * s / m for n, s, m in zip(gi.dims, gi.spacing, dd))
    od = tuple(o - s / 2 + sd / 2 for o, s, sd in zip(gi.origin, gi.spacing, hd))
    return Grid3(tuple(dd), hd, od)


def save(name, **kw):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **kw)
    print(f"wrote {path} ({os.path.getsize(path)} B, {len(kw)} arrays)")


def transfer_cases():
    rng = np.random.default_rng(12345)
    out = {}
    pairs = [random_pair(rng) for _ in range(12)]
    pairs += [
        (def_like(Grid3((17, 13, 11), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0)), (5, 4, 3)),
         Grid3((17, 13, 11), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))),
        (multilevel.deformation_grid_for(Grid3((32, 24, 20), (1.0, 1.5, 2.0), (1.0, -2.0, 0.5)), 4),
         Grid3((32, 24, 20), (1.0, 1.5, 2.0), (1.0, -2.0, 0.5))),
        (def_like(Grid3((26, 26, 26), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0)), (13, 13, 13)),
         Grid3((26, 26, 26), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))),
    ]
    for k, (gd, gi) in enumerate(pairs):
        plan = transfer.build_gather_plan(gd, gi)
        out[f"{k}_gd"] = garr(gd)
        out[f"{k}_gi"] = garr(gi)
        for a in range(3):
            i0, w1 = transfer._axis_transfer(gi, gd, a)
            out[f"{k}_i0_{a}"] = i0.astype(np.int64)
            out[f"{k}_w1_{a}"] = w1
            ap = plan.axes[a]
            out[f"{k}_start_{a}"] = ap.start.astype(np.int64)
            out[f"{k}_counts_{a}"] = ap.counts.astype(np.int64)
            out[f"{k}_weights_{a}"] = ap.weights
        y64 = make_identity(gd).field + rng.standard_normal((3,) + gd.shape)
        r64 = rng.standard_normal((3,) + gi.shape)
        for p, dt in DTYPES.items():
            y = DeformationField(gd, y64.astype(dt))
            r = VectorField3(gi, r64.astype(dt))
            out[f"{k}_y_{p}"] = y.field
            out[f"{k}_r_{p}"] = r.field
            out[f"{k}_P_{p}"] = transfer.apply_P(y, gi).field
            out[f"{k}_Pt_{p}"] = transfer.apply_Pt_gather(r, plan).field
            # the other two P^T variants (transfer.py:199-256), one worker
            out[f"{k}_Pts_{p}"] = transfer.apply_Pt_scatter_atomic(r, gd).field
            out[f"{k}_Ptrb_{p}"] = transfer.apply_Pt_redblack(r, gd).field
    out["n"] = np.array(len(pairs))
    save("transfer", **out)


def warp_cases():
    rng = np.random.default_rng(777)
    out = {}
    cases = [
        (Grid3((9, 8, 7), (1.1, 0.9, 1.3), (0.0, 0.0, 0.0)), 0.8),
        (Grid3((6, 5, 4), (0.8, 1.1, 1.5), (-2.0, 1.0, 0.5)), 2.5),   # many samples outside
        (Grid3((5, 4, 1), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0)), 0.6),    # degenerate z
        (Grid3((1, 6, 5), (1.0, 2.0, 0.5), (3.0, 0.0, 0.0)), 0.6),    # degenerate x
    ]
    for k, (g, amp) in enumerate(cases):
        Tv = synthetic.smooth_random_volume(g, seed=3 + k).values
        yf = synthetic.smooth_random_field(g, seed=4 + k, amplitude_mm=amp).field
        yf[0, 0, 0, 0] = -10.0  # force one sample outside the hull
        s = rng.standard_normal(g.shape)
        out[f"{k}_g"] = garr(g)
        for p, dt in DTYPES.items():
            T = Image3(g, Tv.astype(dt))
            yh = VectorField3(g, yf.astype(dt))
            res = warp.warp_image(T, yh)
            out[f"{k}_T_{p}"] = T.values
            out[f"{k}_yhat_{p}"] = yh.field
            out[f"{k}_s_{p}"] = s.astype(dt)
            out[f"{k}_W_{p}"] = res.warped.values
            out[f"{k}_mask_{p}"] = res.inside_mask
            out[f"{k}_Jt_{p}"] = warp.warp_jacobian_apply_transpose(T, yh, s.astype(dt)).field
            out[f"{k}_G_{p}"] = warp.image_gradient(T).field
            q = VectorField3(g, np.stack([s, -0.5 * s, 2.0 * s]).astype(dt))
            out[f"{k}_q_{p}"] = q.field
            out[f"{k}_Gt_{p}"] = warp.image_gradient_apply_transpose(q, g)
    out["n"] = np.array(len(cases))
    save("warp", **out)


def ngf_cases():
    out = {}
    cases = [
        (Grid3((24, 24, 24), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0)), 4, None),
        (Grid3((19, 17, 13), (1.2, 0.9, 1.5), (-3.0, 2.0, 1.0)), 4, None),
        (Grid3((17, 17, 17), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0)), None, (9, 9, 9)),  # 65^3-on-128^3 style
        (Grid3((16, 16, 16), (2.0, 2.0, 2.0), (0.0, 0.0, 0.0)), 2, None),
    ]
    for k, (gi, ratio, dd) in enumerate(cases):
        gd = multilevel.deformation_grid_for(gi, ratio) if ratio else def_like(gi, dd)
        Rv = synthetic.smooth_random_volume(gi, seed=10 + k).values
        Tv = synthetic.smooth_random_volume(gi, seed=20 + k).values
        yf = synthetic.smooth_random_field(gd, seed=30 + k, amplitude_mm=2.0).field
        out[f"{k}_gi"] = garr(gi)
        out[f"{k}_gd"] = garr(gd)
        for p, dt in DTYPES.items():
            R = Image3(gi, Rv.astype(dt))
            T = Image3(gi, Tv.astype(dt))
            y = DeformationField(gd, yf.astype(dt))
            params = ngf.NgfParams(10.0, 10.0)
            ref = ngf.precompute_reference_terms(R, params)
            plan = transfer.build_gather_plan(gd, gi)
            D, gD = ngf.distance_and_gradient(y, ref, T, plan, params)
            obj = LevelObjective(template=T, ref=ref, plan=plan, params=params, alpha=1.0)
            J, gJ = obj(y.field.ravel())
            out[f"{k}_R_{p}"] = R.values
            out[f"{k}_T_{p}"] = T.values
            out[f"{k}_y_{p}"] = y.field
            out[f"{k}_gR_{p}"] = ref.grad.field
            out[f"{k}_nR_{p}"] = ref.norm
            out[f"{k}_D_{p}"] = np.array(D)
            out[f"{k}_gD_{p}"] = gD.field
            out[f"{k}_J_{p}"] = np.array(J)
            out[f"{k}_Jd_{p}"] = np.array(obj.last_D)
            out[f"{k}_Js_{p}"] = np.array(obj.last_S)
            out[f"{k}_gJ_{p}"] = gJ
            # the objective with the red-black P^T (objective.py:22-60 pt_variant)
            obj_rb = LevelObjective(template=T, ref=ref, plan=plan, params=params, alpha=1.0,
                                    pt_variant="redblack")
            Jrb, gJrb = obj_rb(y.field.ravel())
            out[f"{k}_Jrb_{p}"] = np.array(Jrb)
            out[f"{k}_gJrb_{p}"] = gJrb
    # closed-form orthogonal ramps (tests/test_ngf.py:35-46)
    g = Grid3((6, 6, 6), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    x = g.axis_centers(0)[None, None, :]
    yy = g.axis_centers(1)[None, :, None]
    T = Image3(g, x + np.zeros(g.shape))
    R = Image3(g, yy + np.zeros(g.shape))
    params = ngf.NgfParams(0.1, 0.1)
    ref = ngf.precompute_reference_terms(R, params)
    out["ramp_D"] = np.array(ngf.ngf_value(warp.warp_image(T, make_identity(g)), ref, params,
                                           g.cell_volume))
    out["n"] = np.array(len(cases))
    save("ngf", **out)


def curvature_cases():
    out = {}
    g = Grid3((7, 6, 5), (1.0, 0.9, 1.4), (0.0, 0.0, 0.0))
    g2 = Grid3((6, 6, 2), (1.0, 1.0, 1.0), (0.5, 0.0, 0.0))
    for k, gg in enumerate((g, g2)):
        yf = synthetic.smooth_random_field(gg, seed=9 + k, amplitude_mm=0.7).field
        out[f"{k}_g"] = garr(gg)
        for p, dt in DTYPES.items():
            y = DeformationField(gg, yf.astype(dt))
            out[f"{k}_y_{p}"] = y.field
            out[f"{k}_S_{p}"] = np.array(curvature.curvature_value(y))
            out[f"{k}_gS_{p}"] = curvature.curvature_gradient(y)
            u = y.displacement()[0]
            out[f"{k}_L_{p}"] = curvature.apply_laplacian(u, gg)
            out[f"{k}_LT_{p}"] = curvature.apply_laplacian_transpose(u, gg)
    out["n"] = np.array(2)
    save("curvature", **out)


def multilevel_cases():
    out = {}
    g = Grid3((7, 8, 5), (1.0, 1.2, 2.0), (0.3, -1.0, 2.5))
    v = synthetic.smooth_random_volume(g, seed=1).values
    for p, dt in DTYPES.items():
        img = Image3(g, v.astype(dt))
        pyr = multilevel.build_pyramid(img, 3)
        out[f"pyr_in_{p}"] = img.values
        for k, lv in enumerate(pyr):
            out[f"pyr_{k}_{p}"] = lv.values
            out[f"pyr_{k}_g"] = garr(lv.grid)
    g2 = Grid3((33, 20, 17), (0.7, 1.0, 1.3), (0.0, 5.0, -2.0))
    v2 = synthetic.smooth_random_volume(g2, seed=2).values
    for p, dt in DTYPES.items():
        img = Image3(g2, v2.astype(dt))
        ds = multilevel.downsample_image(img)
        out[f"ds_in_{p}"] = img.values
        out[f"ds_out_{p}"] = ds.values
    out["ds_g_in"] = garr(g2)
    out["ds_g_out"] = garr(multilevel.downsample_image(Image3(g2, v2)).grid)
    # auto levels and def grids (tests/test_multilevel.py:49-70)
    dims_list = [(64, 64, 64), (16, 16, 16), (256, 256, 128), (30, 17, 9), (8, 8, 1), (512, 512, 512)]
    out["auto_dims"] = np.array(dims_list)
    out["auto_levels"] = np.array([multilevel.num_auto_levels(d, 16) for d in dims_list])
    gdefs = [Grid3((30, 17, 9), (1.0, 1.5, 2.0), (1.0, 2.0, 3.0)), Grid3((8, 8, 1), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0)),
             Grid3((256, 256, 256), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0)), Grid3((128, 128, 128), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))]
    for k, gi in enumerate(gdefs):
        for ratio in (2, 4, 8):
            out[f"defgrid_{k}_{ratio}"] = garr(multilevel.deformation_grid_for(gi, ratio))
        out[f"defgrid_{k}_gi"] = garr(gi)
    # prolongation (tests/test_multilevel.py:73-109)
    img = Grid3((16, 12, 8), (1.0, 1.3, 2.0), (0.0, 0.0, 0.0))
    coarse = multilevel.deformation_grid_for(img, 8)
    fine = multilevel.deformation_grid_for(img, 2)
    yc = synthetic.smooth_random_field(coarse, seed=5, amplitude_mm=1.5).field
    out["pro_gc"] = garr(coarse)
    out["pro_gf"] = garr(fine)
    for p, dt in DTYPES.items():
        y = DeformationField(coarse, yc.astype(dt))
        out[f"pro_in_{p}"] = y.field
        out[f"pro_out_{p}"] = multilevel.prolong_deformation(y, fine).field
    save("multilevel", **out)


def lbfgs_cases():
    out = {}
    rng = np.random.default_rng(4242)
    n = 40
    hist = []
    for _ in range(5):
        s = rng.standard_normal(n)
        y = s + 0.3 * rng.standard_normal(n)
        hist.append((s, y))
    g = rng.standard_normal(n)
    for p, dt in DTYPES.items():
        h = [(s.astype(dt), y.astype(dt)) for s, y in hist]
        out[f"tl_g_{p}"] = g.astype(dt)
        for k, (s, y) in enumerate(h):
            out[f"tl_s{k}_{p}"] = s
            out[f"tl_y{k}_{p}"] = y
        out[f"tl_d_{p}"] = lbfgs.two_loop_direction(h, g.astype(dt))
    # quadratic problem (tests/test_lbfgs.py:11-24)
    Q = rng.standard_normal((12, 12))
    A = Q.T @ Q + 12 * np.eye(12)
    b = rng.standard_normal(12)

    def f(x):
        return 0.5 * float(x @ (A @ x)) - float(b @ x), A @ x - b

    x, tr = lbfgs.lbfgs_minimize(f, np.zeros(12))
    out["quad_A"], out["quad_b"], out["quad_x"] = A, b, x
    out["quad_recs"] = np.array([[r.iteration, r.J, r.grad_inf, r.step, r.ls_evals] for r in tr.records])
    out["quad_reason"] = np.array(tr.stop_reason)
    save("lbfgs", **out)


def register_cases():
    out = {}
    g = Grid3((24, 24, 24), (1.5, 1.5, 1.5), (0.0, 0.0, 0.0))
    center = tuple(o + e / 2 for o, e in zip(g.origin, g.extent))
    R, T = synthetic.make_registration_pair(
        g, synthetic.gaussian_bump_mapping(center, sigma_mm=9.0, amplitude_mm=(2.5, -2.0, 1.5)))
    out["g"] = garr(g)
    out["R"], out["T"] = R.values, T.values
    for p in DTYPES:
        cfg = multilevel.MultilevelConfig(coarsest_min_dim=8, precision=p,
                                          lbfgs=lbfgs.LbfgsConfig(max_iterations=30))
        y, rep = register_run(R, T, cfg)
        out[f"y_{p}"] = y.field
        out[f"gd_{p}"] = garr(y.grid)
        out[f"iters_{p}"] = np.array([lv.iterations for lv in rep.levels])
        out[f"reasons_{p}"] = np.array([lv.stop_reason for lv in rep.levels])
        out[f"J_{p}"] = np.array([lv.records[-1].J for lv in rep.levels])
    save("register", **out)


def register_run(R, T, cfg):
    return multilevel.register(R, T, cfg)


def fileio_cases():
    # MetaImage files written by the reference's writer (fileio.py:122-142): the device
    # package must read them back and write byte-identical files
    from ngfreg import fileio

    g = Grid3((6, 5, 4), (0.7, 1.25, 2.5), (-1.5, 0.25, 3.0))
    fileio.write_volume(Image3(g, synthetic.smooth_random_volume(g, seed=1).values.astype(np.float32)),
                        os.path.join(HERE, "fio_vol_f32.mha"))
    gd = Grid3((4, 3, 5), (2.0, 1.5, 2.5), (1.0, -2.0, 0.0))
    fileio.write_deformation(synthetic.smooth_random_field(gd, seed=3, amplitude_mm=1.5),
                             os.path.join(HERE, "fio_def_f64.mha"))
    print("wrote fio_vol_f32.mha, fio_def_f64.mha")


def evaluation_cases():
    # sample_deformation / landmark_error (evaluation.py:39-89)
    from ngfreg import evaluation

    rng = np.random.default_rng(777)
    out = {}
    cases = [Grid3((7, 6, 5), (2.0, 1.5, 2.5), (1.0, -2.0, 0.0)), Grid3((5, 1, 4), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))]
    for k, gd in enumerate(cases):
        y = synthetic.smooth_random_field(gd, seed=40 + k, amplitude_mm=2.0)
        lo = np.array(gd.domain_min) - 2.0
        hi = np.array(gd.domain_min) + np.array(gd.extent) + 2.0
        pts = lo + (hi - lo) * rng.random((50, 3))
        tm = pts + rng.standard_normal((50, 3))
        res = evaluation.landmark_error(y, evaluation.LandmarkSet(pts), evaluation.LandmarkSet(tm), gd)
        out[f"{k}_g"] = garr(gd)
        out[f"{k}_y"] = y.field
        out[f"{k}_pts"] = pts
        out[f"{k}_tm"] = tm
        out[f"{k}_sample"] = evaluation.sample_deformation(y, pts)
        out[f"{k}_per"] = res.per_landmark_mm
        out[f"{k}_mean"] = np.array(res.mean_mm)
        out[f"{k}_std"] = np.array(res.stddev_mm)
        out[f"{k}_outside"] = res.outside_domain
    out["n"] = np.array(len(cases))
    save("evaluation", **out)


if __name__ == "__main__":
    if len(sys.argv) > 1:  # regenerate selected fixtures, e.g. `make_golden.py transfer`
        for name in sys.argv[1:]:
            globals()[name + "_cases"]()
        sys.exit(0)
    transfer_cases()
    warp_cases()
    ngf_cases()
    curvature_cases()
    multilevel_cases()
    lbfgs_cases()
    register_cases()
    fileio_cases()
    evaluation_cases()
