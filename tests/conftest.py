import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: longer CPU-only case")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def grid_from(arr):
    """(dims, spacing, origin) from the 9-vector written by make_golden.garr."""
    from oracle import ngf_oracle as O
    a = np.asarray(arr, dtype=np.float64)
    return O.grid(tuple(int(v) for v in a[:3]), tuple(a[3:6]), tuple(a[6:9]))


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


def cpu_reference_objective(T, R, gd, gi, workers=None):
    """The reference's LevelObjective on host arrays (unmodified ngfreg staged in oracle/_ref
    by oracle/build_ref.py), or the pinned oracle port when it is not staged.  Grids are
    anything with .dims/.spacing/.origin.  Checker only."""
    from oracle import ref as oref
    workers = workers or (os.cpu_count() or 1)
    mod = oref.load()
    if mod is not None:
        from ngfreg import ngf as rngf, objective as robj, transfer as rtr
        from ngfreg.geometry import Grid3, Image3
        g = Grid3(tuple(gi.dims), tuple(gi.spacing), tuple(gi.origin))
        gdr = Grid3(tuple(gd.dims), tuple(gd.spacing), tuple(gd.origin))
        params = rngf.NgfParams(10.0, 10.0)
        ref = rngf.precompute_reference_terms(Image3(g, R), params)
        return robj.LevelObjective(template=Image3(g, T), ref=ref, plan=rtr.build_gather_plan(gdr, g),
                                   params=params, alpha=1.0, workers=workers)
    from oracle import ngf_oracle as O
    return O.Objective(T, R, O.grid(gd.dims, gd.spacing, gd.origin), O.grid(gi.dims, gi.spacing, gi.origin),
                       workers=workers)
