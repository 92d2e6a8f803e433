"""CPU-only checks of the product's host side (no GPU): the C-ABI loads and exports
every declared symbol, the host f64 plans and grid metadata are bit-exact with
the reference fixtures, and argument/grid errors map to the reference's
exception types."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, load_golden

import paper_1812_06765_b200 as ngf
from paper_1812_06765_b200 import _lib


def _g(arr):
    a = np.asarray(arr, dtype=np.float64)
    return ngf.Grid3(tuple(int(v) for v in a[:3]), tuple(a[3:6]), tuple(a[6:9]))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    header = open(os.path.join(ROOT, "include", "ngf_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(ngf_\w+)\s*\(", header, re.M))
    assert len(declared) >= 30
    missing = [n for n in declared if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_lib.EXPORTED) <= declared
    assert lib.ngf_version() >= 100


def test_plans_bit_exact_vs_reference():
    z = load_golden("transfer")
    for k in range(int(z["n"])):
        gd, gi = _g(z[f"{k}_gd"]), _g(z[f"{k}_gi"])
        plan = ngf.build_gather_plan(gd, gi)
        for a in range(3):
            i0, w1, st, cnt, w = plan._plan.axis(a)
            assert np.array_equal(i0, z[f"{k}_i0_{a}"])
            assert np.array_equal(w1, z[f"{k}_w1_{a}"])  # f64, bit for bit
            assert np.array_equal(st, z[f"{k}_start_{a}"])
            assert np.array_equal(cnt, z[f"{k}_counts_{a}"])
            assert np.array_equal(w, z[f"{k}_weights_{a}"])
            ap = plan.axes[a]
            assert np.array_equal(ap.weights, z[f"{k}_weights_{a}"])


def test_pyramid_and_def_grid_metadata_bit_exact():
    z = load_golden("multilevel")
    for dims, lv in zip(z["auto_dims"], z["auto_levels"]):
        assert ngf.num_auto_levels(tuple(int(d) for d in dims), 16) == int(lv)
    for k in range(4):
        gi = _g(z[f"defgrid_{k}_gi"])
        for ratio in (2, 4, 8):
            gd = ngf.deformation_grid_for(gi, ratio)
            assert np.array_equal(np.array([*gd.dims, *gd.spacing, *gd.origin]),
                                  z[f"defgrid_{k}_{ratio}"])
    from paper_1812_06765_b200.multilevel import _coarser
    assert np.array_equal(np.array([*_coarser(_g(z["ds_g_in"])).dims,
                                    *_coarser(_g(z["ds_g_in"])).spacing,
                                    *_coarser(_g(z["ds_g_in"])).origin]), z["ds_g_out"])
    g = ngf.Grid3((7, 8, 5), (1.0, 1.2, 2.0), (0.3, -1.0, 2.5))
    for k in (2, 1, 0):
        assert np.array_equal(np.array([*g.dims, *g.spacing, *g.origin]), z[f"pyr_{k}_g"])
        g = _coarser(g)


def test_axis_transfer_degenerate_and_prolong_maps():
    gi = ngf.Grid3((8, 8, 1), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    gd = ngf.deformation_grid_for(gi, 4)
    assert gd.dims == (2, 2, 1)
    i0, w1 = ngf.transfer.axis_transfer(gi, gd, 2)
    assert i0.tolist() == [0] and w1.tolist() == [0.0]
    # coarse -> fine def grids (no dims ordering constraint for prolongation plans)
    img = ngf.Grid3((16, 12, 8), (1.0, 1.3, 2.0), (0.0, 0.0, 0.0))
    c, f = ngf.deformation_grid_for(img, 8), ngf.deformation_grid_for(img, 2)
    from oracle import ngf_oracle as O
    for a in range(3):
        i0, w1 = ngf.transfer.axis_transfer(f, c, a)
        oi0, ow1 = O.axis_transfer(O.grid(f.dims, f.spacing, f.origin),
                                   O.grid(c.dims, c.spacing, c.origin), a)
        assert np.array_equal(i0, oi0) and np.array_equal(w1, ow1)


def test_grid_errors_match_reference_types():
    gi = ngf.Grid3((4, 4, 4), (1, 1, 1), (0, 0, 0))
    bad = ngf.Grid3((2, 2, 2), (2, 2, 2), (10, 0, 0))
    with pytest.raises(ngf.GridError):
        ngf.build_gather_plan(bad, gi)
    with pytest.raises(ngf.GridError):
        ngf.Grid3((0, 1, 1), (1, 1, 1), (0, 0, 0))
    with pytest.raises(ngf.GridError):
        ngf.Grid3((1, 1, 1), (1, -1, 1), (0, 0, 0))
    with pytest.raises(ngf.GridError):
        ngf.Image3(gi, np.zeros((4, 4, 3)))
    with pytest.raises(ngf.GridError):
        ngf.Image3(gi, np.full((4, 4, 4), np.nan))
    # the C-ABI reports the same conditions as codes
    p = ctypes.c_void_p()
    rc = _lib.lib().ngf_plan_create(ctypes.byref(_lib.ngf_grid(bad)), ctypes.byref(_lib.ngf_grid(gi)),
                                    ctypes.byref(p))
    assert rc == _lib.NGF_EGRID
    with pytest.raises(ngf.GridError):
        _lib.check(rc, "plan")


def test_config_validation():
    with pytest.raises(ValueError):
        ngf.MultilevelConfig(num_levels=0)
    with pytest.raises(ValueError):
        ngf.MultilevelConfig(alpha=0.0)
    with pytest.raises(ValueError):
        ngf.MultilevelConfig(grid_ratio=0)
    with pytest.raises(ValueError):
        ngf.LbfgsConfig(memory=0)
    with pytest.raises(ValueError):
        ngf.LbfgsConfig(c1=1.5)
    with pytest.raises(ValueError):
        ngf.StoppingRules(tol_J=0.0)
    with pytest.raises(ValueError):
        ngf.NgfParams(tau=0.0)
    with pytest.raises(ValueError):
        ngf.precision_dtype("f16")


def test_synthetic_inputs_match_reference_generators():
    """The package's restated generators (used on the GPU box) produce the oracle's bytes."""
    from oracle import ngf_oracle as O
    g = ngf.Grid3((9, 8, 7), (1.1, 0.9, 1.3), (0.0, 0.0, 0.0))
    og = O.grid(g.dims, g.spacing, g.origin)
    assert np.array_equal(ngf.smooth_random_volume(g, seed=3).values, O.smooth_random_volume(og, 3))
    assert np.array_equal(ngf.smooth_random_field(g, seed=4, amplitude_mm=0.8).field,
                          O.smooth_random_field(og, 4, 0.8))
    m = ngf.gaussian_bump_mapping((5, 4, 3), 3.0, (1.0, -0.5, 0.25))
    R, T = ngf.make_registration_pair(g, m)
    Ro, To = O.registration_pair(og, O.bump_mapping((5, 4, 3), 3.0, (1.0, -0.5, 0.25)))
    assert np.array_equal(R.values, Ro) and np.array_equal(T.values, To)


def test_ct_phantom_is_deterministic_and_ct_like():
    R, T, _ = ngf.ct_pair(32, seed=0)
    R2, T2, _ = ngf.ct_pair(32, seed=0)
    assert np.array_equal(R.values, R2.values) and np.array_equal(T.values, T2.values)
    v = T.values
    assert v.min() < -900 and v.max() > 300  # air and bone present
    assert np.abs(R.values - T.values).max() > 10  # the pair actually differs


def test_unknown_pt_variant_is_a_value_error():
    # transfer.py:259-266 / objective.py: unknown variant names raise ValueError
    with pytest.raises(ValueError):
        ngf.LevelObjective(template=None, ref=None, plan=None, params=None, alpha=1.0,
                           pt_variant="bogus")
