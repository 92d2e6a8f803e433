"""Full multilevel registration on the device vs the reference (multilevel.py:179-247).

Parity protocol: report max-abs displacement difference over
all deformation nodes and over the interior (>= 2 def cells from every face),
plus per-level iteration counts; the bar is 0.05 voxel on the interior.  The
exact pipeline must also reproduce the reference's accepted iterates."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

import paper_1812_06765_b200 as ngf  # noqa: E402
from oracle import ngf_oracle as O  # noqa: E402

BAR_VOXEL = 0.05


def _g(arr):
    a = np.asarray(arr, dtype=np.float64)
    return ngf.Grid3(tuple(int(v) for v in a[:3]), tuple(a[3:6]), tuple(a[6:9]))


def _field_stats(y, y_ref, gd, voxel):
    d = np.sqrt(np.sum((y.astype(np.float64) - y_ref.astype(np.float64)) ** 2, axis=0)) / voxel
    inner = d[2:-2, 2:-2, 2:-2] if min(gd.shape) > 4 else d
    return float(d.max()), float(inner.max()), float(d.mean())


@pytest.mark.parametrize("p", ["f32", "f64"])
def test_register_matches_reference_fixture(p):
    z = load_golden("register")
    g = _g(z["g"])
    cfg = ngf.MultilevelConfig(coarsest_min_dim=8, precision=p,
                               lbfgs=ngf.LbfgsConfig(max_iterations=30))
    R, T = ngf.Image3(g, z["R"]), ngf.Image3(g, z["T"])
    y, rep = ngf.register(R, T, cfg)
    gd = _g(z[f"gd_{p}"])
    assert y.grid == gd and y.field.dtype == np.dtype(p.replace("f", "float"))
    mx, inner, mean = _field_stats(y.field, z[f"y_{p}"], gd, g.spacing[0])
    iters = [lv.iterations for lv in rep.levels]
    print(f"{p}: iterations {iters} vs ref {list(z[f'iters_{p}'])}; max {mx:.4f} "
          f"interior {inner:.4f} mean {mean:.5f} voxel")
    assert inner <= BAR_VOXEL
    # exact pipeline: bit-exact J and gradients; the trajectory still differs through the
    # L-BFGS dot products (double-accumulated here, BLAS sdot/ddot in the reference)
    y2, rep2 = ngf.register(R, T, ngf.MultilevelConfig(coarsest_min_dim=8, precision=p, exact=True,
                                                        lbfgs=ngf.LbfgsConfig(max_iterations=30)))
    mx2, inner2, _ = _field_stats(y2.field, z[f"y_{p}"], gd, g.spacing[0])
    print(f"{p} exact: iterations {[lv.iterations for lv in rep2.levels]}; max {mx2:.4f} "
          f"interior {inner2:.4f}")
    assert rep2.levels[0].iterations == int(z[f"iters_{p}"][0])
    assert inner2 <= BAR_VOXEL


def test_register_c1_vs_oracle():
    """Config 1: 64^3 Gaussian-bump pair, single level, f32."""
    g = ngf.Grid3((64, 64, 64), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    center = tuple(o + e / 2 for o, e in zip(g.origin, g.extent))
    mapping = ngf.gaussian_bump_mapping(center, 18.0, (3.0, -2.0, 1.5))
    R, T = ngf.make_registration_pair(g, mapping)
    y, rep = ngf.register(R, T, ngf.MultilevelConfig(num_levels=1, precision="f32"))
    y_ref, gd, info = O.register(R.values, T.values, O.grid(g.dims), num_levels=1, precision="f32",
                                 workers=8)
    mx, inner, mean = _field_stats(y.field, y_ref, y.grid, 1.0)
    print(f"C1: iterations {rep.levels[0].iterations} vs oracle {info[0]['iterations']}; "
          f"max {mx:.4f} interior {inner:.4f} mean {mean:.5f} voxel")
    assert inner <= BAR_VOXEL
    # recovery against the known mapping (tests/test_acceptance.py:303-316)
    pts = ngf.probe_lattice(g, n_per_axis=5, margin=0.25)
    truth = np.stack(mapping(pts[:, 0], pts[:, 1], pts[:, 2]), axis=1)
    from paper_1812_06765_b200.geometry import DeformationField
    mapped = O_sample(y.field.astype(np.float64), y.grid, pts)
    err = np.linalg.norm(mapped - truth, axis=1).mean()
    assert err < 0.5


def O_sample(field, grid, pts):
    """Trilinear clamp-to-edge evaluation of a deformation at world points
    (evaluation.py:39-65 of the reference; host-side scoring only)."""
    out = np.zeros((len(pts), 3))
    idx, fr = [], []
    for a in range(3):
        t = (pts[:, a] - grid.origin[a]) / grid.spacing[a]
        n = grid.dims[a]
        i0 = np.clip(np.floor(t).astype(int), 0, max(n - 2, 0))
        idx.append(i0)
        fr.append(np.clip(t - i0, 0, 1) if n > 1 else np.zeros(len(pts)))
    for dz in (0, 1):
        for dy in (0, 1):
            for dx in (0, 1):
                w = ((fr[0] if dx else 1 - fr[0]) * (fr[1] if dy else 1 - fr[1])
                     * (fr[2] if dz else 1 - fr[2]))
                ix = np.minimum(idx[0] + dx, grid.dims[0] - 1)
                iy = np.minimum(idx[1] + dy, grid.dims[1] - 1)
                iz = np.minimum(idx[2] + dz, grid.dims[2] - 1)
                out += w[:, None] * field[:, iz, iy, ix].T
    return out


def test_register_identical_images_stays_near_identity():
    g = ngf.Grid3((16, 16, 16), (2.0, 2.0, 2.0), (0.0, 0.0, 0.0))
    T = ngf.smooth_random_volume(g, seed=8)
    y, _ = ngf.register(T, T, ngf.MultilevelConfig(coarsest_min_dim=8,
                                                   lbfgs=ngf.LbfgsConfig(max_iterations=10)))
    pts = ngf.probe_lattice(g, n_per_axis=5, margin=0.25)
    drift = np.linalg.norm(O_sample(y.field, y.grid, pts) - pts, axis=1)
    assert drift.mean() < 1.0 and drift.max() < 2.0


def test_register_rejects_mismatched_grids():
    R = ngf.smooth_random_volume(ngf.Grid3((8, 8, 8), (1, 1, 1), (0, 0, 0)), seed=1)
    T = ngf.smooth_random_volume(ngf.Grid3((9, 8, 8), (1, 1, 1), (0, 0, 0)), seed=2)
    with pytest.raises(ngf.GridError):
        ngf.register(R, T)


@pytest.mark.parametrize("exact", [False, True])
def test_native_driver_matches_python_driver(monkeypatch, exact):
    """ngf_lbfgs_run_level (native loop) takes the Python driver's decisions: identical
    iteration records, (J, D, S) rows, stop reason, evaluation count and final field."""
    import torch

    gi = ngf.Grid3((40, 36, 32), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    gd = ngf.deformation_grid_for(gi, 4)
    R = ngf.smooth_random_volume(gi, seed=11).values.astype(np.float32)
    T = ngf.smooth_random_volume(gi, seed=12).values.astype(np.float32)
    x0 = ngf.make_identity(gd).field.astype(np.float32).ravel()
    plan = ngf.build_gather_plan(gd, gi)
    out = []
    for py in (True, False):
        if py:
            monkeypatch.setenv("NGF_PY_LBFGS", "1")
        else:
            monkeypatch.delenv("NGF_PY_LBFGS", raising=False)
        obj = ngf.LevelObjective.from_device(torch.from_numpy(T).cuda(), torch.from_numpy(R).cuda(), plan,
                                             ngf.NgfParams(), 1.0, exact=exact)
        x, tr = ngf.lbfgs_minimize(obj, x0.copy(), ngf.LbfgsConfig(max_iterations=25))
        out.append((x, tr))
    (xp, tp), (xn, tn) = out
    assert tn.stop_reason == tp.stop_reason and tn.evaluations == tp.evaluations
    assert [(r.J, r.grad_inf, r.step, r.ls_evals) for r in tn.records] == \
           [(r.J, r.grad_inf, r.step, r.ls_evals) for r in tp.records]
    assert tn.J_rows == tp.J_rows
    assert np.array_equal(xn, xp)


@pytest.mark.parametrize("cfg", [
    ngf.LbfgsConfig(max_iterations=30),
    ngf.LbfgsConfig(memory=1, max_iterations=20),                        # history ageing
    ngf.LbfgsConfig(initial_step=40.0, max_ls_steps=3, max_iterations=20),  # backtracking, failure
    ngf.LbfgsConfig(initial_step=0.05, step_shrink=0.7, max_iterations=12),  # long forward expansions
], ids=["default", "memory1", "backtrack", "expand"])
def test_graph_driver_matches_host_and_python(monkeypatch, cfg):
    """The graph-driven level loop (csrc/solver_graph.cu: one CUDA graph, device-side
    decisions) and the host-driven native loop take exactly the Python driver's decisions."""
    import torch

    from paper_1812_06765_b200._lib import lib

    gi = ngf.Grid3((40, 36, 32), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    gd = ngf.deformation_grid_for(gi, 4)
    R = ngf.smooth_random_volume(gi, seed=21).values.astype(np.float32)
    T = ngf.smooth_random_volume(gi, seed=22).values.astype(np.float32)
    x0 = ngf.make_identity(gd).field.astype(np.float32).ravel()
    plan = ngf.build_gather_plan(gd, gi)
    out = []
    try:
        for mode in ("python", "host", "graph"):
            if mode == "python":
                monkeypatch.setenv("NGF_PY_LBFGS", "1")
            else:
                monkeypatch.delenv("NGF_PY_LBFGS", raising=False)
                lib().ngf_lbfgs_set_graph(1 if mode == "graph" else 0)
            obj = ngf.LevelObjective.from_device(torch.from_numpy(T).cuda(), torch.from_numpy(R).cuda(), plan,
                                                 ngf.NgfParams(), 1.0)
            runs = lib().ngf_lbfgs_graph_runs()
            out.append(ngf.lbfgs_minimize(obj, x0.copy(), cfg))
            assert lib().ngf_lbfgs_graph_runs() - runs == (1 if mode == "graph" else 0), mode
    finally:
        lib().ngf_lbfgs_set_graph(0)
    xp, tp = out[0]
    for x, t in out[1:]:
        assert (t.stop_reason, t.evaluations, t.iterations, t.line_search_failed) == \
               (tp.stop_reason, tp.evaluations, tp.iterations, tp.line_search_failed)
        assert [(r.J, r.grad_inf, r.step, r.ls_evals) for r in t.records] == \
               [(r.J, r.grad_inf, r.step, r.ls_evals) for r in tp.records]
        assert t.J_rows == tp.J_rows
        assert np.array_equal(x, xp)


def test_native_driver_edge_cases(monkeypatch):
    """Stationary start (constant images at the identity: grad J = 0 exactly) and a zero
    iteration budget give the same traces from the native and the Python drivers."""
    import torch

    gi = ngf.Grid3((24, 20, 16), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    gd = ngf.deformation_grid_for(gi, 4)
    x0 = ngf.make_identity(gd).field.astype(np.float32).ravel()
    plan = ngf.build_gather_plan(gd, gi)
    flat = np.full(gi.shape, 100.0, dtype=np.float32)
    cases = ((flat, flat, ngf.LbfgsConfig(), "stationary start"),
             (ngf.smooth_random_volume(gi, seed=4).values.astype(np.float32),
              ngf.smooth_random_volume(gi, seed=3).values.astype(np.float32), ngf.LbfgsConfig(max_iterations=0),
              "max iterations"))
    for T, R, cfg, reason in cases:
        out = []
        for py in (True, False):
            if py:
                monkeypatch.setenv("NGF_PY_LBFGS", "1")
            else:
                monkeypatch.delenv("NGF_PY_LBFGS", raising=False)
            obj = ngf.LevelObjective.from_device(torch.from_numpy(T).cuda(), torch.from_numpy(R).cuda(), plan,
                                                 ngf.NgfParams(), 1.0)
            out.append(ngf.lbfgs_minimize(obj, x0.copy(), cfg))
        (xp, tp), (xn, tn) = out
        assert tn.stop_reason == tp.stop_reason == reason and tn.evaluations == tp.evaluations
        assert tn.iterations == tp.iterations == 0 and tn.J_rows == tp.J_rows
        assert np.array_equal(xn, xp) and np.array_equal(xn, x0)


@pytest.mark.parametrize("exact", [False, True])
def test_concurrent_registrations_on_streams_match_sequential(exact):
    """Config 4 on one GPU: registrations in flight on several host threads, one CUDA
    stream each (levels of different sizes created concurrently, per-stream reduction
    scratch, table uploads that must land before another stream's kernels read them)
    give bit-identical fields to the same registrations run one after another."""
    import threading

    import torch

    cfg = ngf.MultilevelConfig(num_levels=3, grid_ratio=4, precision="f32", exact=exact,
                               lbfgs=ngf.LbfgsConfig(max_iterations=8))
    n = 64 if exact else 128
    pairs = [ngf.ct_pair(n, seed=500 + p, dtype=np.float32)[:2] for p in range(6)]
    ref = [ngf.register(R, T, cfg)[0].field for R, T in pairs]
    k = 3
    streams = [torch.cuda.Stream() for _ in range(k)]
    out = [None] * len(pairs)
    errors = []

    def work(i):
        try:
            with torch.cuda.stream(streams[i]):
                for j in range(i, len(pairs), k):
                    out[j] = ngf.register(*pairs[j], cfg)[0].field
                streams[i].synchronize()
        except Exception as e:  # re-raised below
            errors.append(e)

    threads = [threading.Thread(target=work, args=(i,)) for i in range(k)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    torch.cuda.synchronize()
    assert not errors, errors[0]
    for o, r in zip(out, ref):
        assert np.array_equal(o, r)
