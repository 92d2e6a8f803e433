"""Full-registration fixtures at the BASELINE configs, from the REAL reference (build container only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_large.py [c2] [c3]

Runs `ngfreg.multilevel.register` (/root/reference/pkg/src, read-only) on the
synthetic CT-shaped pairs of bench.py / SURVEY.md §8(d):
  * C2: 128^3, 3 levels, grid ratio 2 (64^3 finest deformation grid), f32 and f64;
  * C3: 256^3, 4 levels, grid ratio 4 (64^3 finest deformation grid), f32.
The pairs come from `paper_1812_06765_b200.synthetic.ct_pair` (host numpy, no device);
the fixture stores a SHA-256 of R and T so the GPU test can prove it rebuilt the same
bytes.  Stored per case: the final field (as float32 for both precisions: ample for a
0.05-voxel bar, and half the fixture size), per-level iterations / stop reasons, the
accepted-iterate J trace of every level, the
reference's probe error against the known mapping (synthetic.py:72-80 lattice,
evaluation.py:68-90 style mean/max) and the reference's wall time on this host.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

from ngfreg import multilevel  # noqa: E402
from ngfreg.evaluation import sample_deformation  # noqa: E402
from ngfreg.geometry import Grid3, Image3  # noqa: E402
from ngfreg.lbfgs import LbfgsConfig, StoppingRules  # noqa: E402
from ngfreg.synthetic import probe_lattice  # noqa: E402

from paper_1812_06765_b200.synthetic import ct_pair  # noqa: E402  (host numpy only)

CASES = {
    # name: (n, levels, ratio, precisions, fixed iteration budget or False)
    "c2": (128, 3, 2, ("f32", "f64"), False),
    "c3": (256, 4, 4, ("f32",), False),
    # the same pairs with the stopping tolerances switched off (1e-12) and a fixed iteration
    # budget per level, so both sides run the same number of iterations towards the minimiser
    # and the final field no longer depends on when a tolerance fires
    "c2conv": (128, 3, 2, ("f32",), 300),
    "c3conv": (256, 4, 4, ("f32",), 100),
}
CONVERGED_TOL = 1e-12


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def run(name: str, workers: int):
    n, levels, ratio, precs, conv = CASES[name]
    R, T, mapping = ct_pair(n, seed=0)
    g = Grid3(R.grid.dims, R.grid.spacing, R.grid.origin)
    out = {"R_sha": np.array(sha(R.values)), "T_sha": np.array(sha(T.values)),
           "n": np.array(n), "levels": np.array(levels), "ratio": np.array(ratio),
           "workers": np.array(workers), "converged": np.array(bool(conv)),
           "tol": np.array(CONVERGED_TOL if conv else -1.0),
           "max_iterations": np.array(conv if conv else 100)}
    pts = probe_lattice(g, n_per_axis=7, margin=0.2)
    truth = np.stack(mapping(pts[:, 0], pts[:, 1], pts[:, 2]), axis=1)
    for p in precs:
        kw = {}
        if conv:
            kw = dict(lbfgs=LbfgsConfig(max_iterations=conv),
                      stopping=StoppingRules(tol_J=CONVERGED_TOL, tol_grad=CONVERGED_TOL,
                                             tol_step=CONVERGED_TOL))
        cfg = multilevel.MultilevelConfig(num_levels=levels, grid_ratio=ratio, precision=p,
                                          workers=workers, **kw)
        t0 = time.perf_counter()
        y, rep = multilevel.register(Image3(g, R.values), Image3(g, T.values), cfg)
        dt = time.perf_counter() - t0
        err = np.linalg.norm(sample_deformation(y, pts) - truth, axis=1)
        out[f"y_{p}"] = y.field.astype(np.float32)  # ample for a 0.05-voxel bar
        out[f"gd_{p}"] = np.array([*y.grid.dims, *y.grid.spacing, *y.grid.origin])
        out[f"iters_{p}"] = np.array([lv.iterations for lv in rep.levels])
        out[f"stops_{p}"] = np.array([lv.stop_reason for lv in rep.levels])
        for li, lv in enumerate(rep.levels):  # accepted-iterate objective per level (trajectory)
            out[f"Jtrace_{p}_{li}"] = np.array([r.J for r in lv.records], dtype=np.float64)
        out[f"probe_mean_{p}"] = np.array(err.mean())
        out[f"probe_max_{p}"] = np.array(err.max())
        out[f"seconds_{p}"] = np.array(dt)
        print(f"{name} {p}: {dt:.1f} s on {workers} workers, iterations "
              f"{[lv.iterations for lv in rep.levels]}, stops {[lv.stop_reason for lv in rep.levels]}, "
              f"probe error mean {err.mean():.4f} max {err.max():.4f} mm", flush=True)
    path = os.path.join(HERE, f"register_{name}.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path)} B)")


if __name__ == "__main__":
    names = [a for a in sys.argv[1:] if a in CASES] or ["c2", "c3"]
    for nm in names:
        run(nm, os.cpu_count() or 1)
