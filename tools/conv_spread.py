"""Spread of equally valid f32 runs of the tolerance-off registrations (c2conv / c3conv):
per level iterations, stop reason and final J, and the probe error, for the build and
variant this process runs (compare against tests/golden/register_<name>.npz).
    python tools/conv_spread.py c3conv"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

import paper_1812_06765_b200 as ngf  # noqa: E402
from paper_1812_06765_b200.evaluation import sample_deformation  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3conv"
z = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                         f"register_{name}.npz"))
n, levels, ratio = int(z["n"]), int(z["levels"]), int(z["ratio"])
R, T, mapping = ngf.ct_pair(n, seed=0, dtype=np.float32)
tol = float(z["tol"])
cfg = ngf.MultilevelConfig(num_levels=levels, grid_ratio=ratio, precision="f32",
                           lbfgs=ngf.LbfgsConfig(max_iterations=int(z["max_iterations"])),
                           stopping=ngf.StoppingRules(tol_J=tol, tol_grad=tol, tol_step=tol),
                           exact=os.environ.get("EXACT") == "1")
y, rep = ngf.register(R, T, cfg)
pts = ngf.probe_lattice(R.grid, n_per_axis=7, margin=0.2)
truth = np.stack(mapping(pts[:, 0], pts[:, 1], pts[:, 2]), axis=1)
err = np.linalg.norm(sample_deformation(y, pts) - truth, axis=1)
d = np.sqrt(np.sum((y.field.astype(np.float64) - z["y_f32"].astype(np.float64)) ** 2, axis=0))
tag = os.environ.get("TAG", "")
print(f"{name} {tag}: probe {err.mean():.4f} (ref {float(z['probe_mean_f32']):.4f}); field diff mean {d.mean():.4f} max {d.max():.4f}")
for i, lv in enumerate(rep.levels):
    Jr = z[f"Jtrace_f32_{i}"]
    Jl = lv.records[-1].J if lv.records else float("nan")
    print(f"  level {i}: {lv.iterations} it, {lv.stop_reason:32s} J_end {Jl:.6f} | ref {len(Jr)} it "
          f"{str(z['stops_f32'][i]):20s} J_end {Jr[-1]:.6f} (rel {(Jl - Jr[-1]) / Jr[-1]:+.2e}); "
          f"ref J at our count {Jr[min(lv.iterations, len(Jr)) - 1]:.6f}")
