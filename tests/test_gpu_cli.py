"""The command line on the GPU (cli.py:120-227) and the device landmark probe
(evaluation.py:39-89): register -> warp -> evaluate round trip, resample, compare
deformations, benchmark; `sample_deformation` bit-identical to the reference."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

import paper_1812_06765_b200 as ngf  # noqa: E402
from paper_1812_06765_b200 import evaluation, fileio  # noqa: E402
from paper_1812_06765_b200.cli import EXIT_OK, main  # noqa: E402


def test_sample_deformation_and_landmark_error_match_reference():
    z = load_golden("evaluation")
    for k in range(int(z["n"])):
        a = z[f"{k}_g"]
        g = ngf.Grid3(tuple(int(v) for v in a[:3]), tuple(a[3:6]), tuple(a[6:9]))
        y = ngf.DeformationField(g, z[f"{k}_y"])
        assert np.array_equal(evaluation.sample_deformation(y, z[f"{k}_pts"]), z[f"{k}_sample"])
        res = evaluation.landmark_error(y, evaluation.LandmarkSet(z[f"{k}_pts"]),
                                        evaluation.LandmarkSet(z[f"{k}_tm"]), g)
        assert np.array_equal(res.per_landmark_mm, z[f"{k}_per"])
        assert res.mean_mm == float(z[f"{k}_mean"]) and res.stddev_mm == float(z[f"{k}_std"])
        assert np.array_equal(res.outside_domain, z[f"{k}_outside"])


@pytest.fixture()
def pair(tmp_path):
    g = ngf.Grid3((16, 16, 16), (2.0, 2.0, 2.0), (0.0, 0.0, 0.0))
    center = tuple(o + e / 2 for o, e in zip(g.origin, g.extent))
    R, T = ngf.make_registration_pair(g, ngf.gaussian_bump_mapping(center, sigma_mm=8.0,
                                                                   amplitude_mm=(1.5, -1.0, 0.5)))
    rp, tp = str(tmp_path / "R.mha"), str(tmp_path / "T.mha")
    fileio.write_volume(R, rp)
    fileio.write_volume(T, tp)
    return g, rp, tp


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_register_warp_evaluate_roundtrip(pair, tmp_path, capsys, precision):
    g, rp, tp = pair
    yp, wp, rep = str(tmp_path / "y.mha"), str(tmp_path / "w.mha"), str(tmp_path / "rep.txt")
    assert main(["register", "--reference", rp, "--template", tp, "--out-deformation", yp, "--out-warped", wp,
                 "--levels", "2", "--max-iter", "25", "--report", rep, "--precision", precision]) == EXIT_OK
    y = fileio.read_deformation(yp)
    assert y.grid.same_extent(g)
    warped = fileio.read_volume(wp)
    assert warped.grid == g
    text = open(rep).read()
    assert "[level 0]" in text and "[level 1]" in text and "iterations" in text
    R = fileio.read_volume(rp).values
    # warping again through the CLI reproduces the register output; difference image
    w2, dp = str(tmp_path / "w2.mha"), str(tmp_path / "d.mha")
    assert main(["warp", "--template", tp, "--deformation", yp, "--out", w2, "--reference", rp,
                 "--out-difference", dp]) == EXIT_OK
    if precision == "f64":
        assert np.array_equal(fileio.read_volume(w2).values, warped.values)
    else:  # register warps in f32, the CLI warp reads the f64 template
        assert np.allclose(fileio.read_volume(w2).values, warped.values, rtol=1e-4, atol=1e-2)
    assert np.allclose(fileio.read_volume(dp).values, fileio.read_volume(w2).values - R)
    # landmark evaluation: the identity reference landmarks vs themselves
    lm = str(tmp_path / "lm.txt")
    open(lm, "w").write("8 8 8\n4 9 12\n")
    capsys.readouterr()
    assert main(["evaluate", "--deformation", yp, "--landmarks-ref", lm, "--landmarks-template", lm,
                 "--image-grid-from", rp, "--frame", "index1"]) == EXIT_OK
    assert "landmark error" in capsys.readouterr().out


def test_resample_and_compare_deformation(tmp_path, capsys):
    g1 = ngf.Grid3((8, 8, 8), (2, 2, 2), (0, 0, 0))
    g2 = ngf.Grid3((10, 10, 10), (1.6, 1.6, 1.6), (0.2, 0.2, 0.2))
    a, b, out = str(tmp_path / "a.mha"), str(tmp_path / "b.mha"), str(tmp_path / "b_on_a.mha")
    fileio.write_volume(ngf.smooth_random_volume(g1, seed=3), a)
    fileio.write_volume(ngf.smooth_random_volume(g2, seed=4), b)
    assert main(["resample", "--input", b, "--like", a, "--out", out]) == EXIT_OK
    assert fileio.read_volume(out).grid == g1
    dg = ngf.deformation_grid_for(g1, 4)
    y1, y2, lm = str(tmp_path / "y1.mha"), str(tmp_path / "y2.mha"), str(tmp_path / "lm.txt")
    fileio.write_deformation(ngf.make_identity(dg), y1)
    fileio.write_deformation(ngf.DeformationField(dg, ngf.make_identity(dg).field + 0.5), y2)
    open(lm, "w").write("8 8 8\n")
    capsys.readouterr()
    assert main(["evaluate", "--deformation", y1, "--landmarks-ref", lm, "--landmarks-template", lm,
                 "--image-grid-from", a, "--frame", "world", "--compare-deformation", y2]) == EXIT_OK
    out = capsys.readouterr().out
    assert "field difference" in out and f"{np.sqrt(0.75):.6e}" in out


def test_benchmark_subcommand(tmp_path):
    out = str(tmp_path / "bench.tsv")
    assert main(["benchmark", "--dims", "12,12,12", "--precision", "f64", "--pt-variant", "gather,redblack",
                 "--reps", "3", "--out", out]) == EXIT_OK
    text = open(out).read()
    assert "redblack" in text and text.count("\n") == 1 + 5


def test_benchmark_checksums_equal_the_reference():
    """The device harness and the reference's (ngfreg.benchmark.run_benchmark, staged in
    oracle/_ref) hash identical results for the exact operators on the same inputs."""
    from oracle import ref as oref
    from paper_1812_06765_b200.benchmark import run_benchmark
    mod = oref.load()
    if mod is None:
        pytest.skip("reference not staged (oracle/build_ref.py)")
    from ngfreg import benchmark as rb
    kw = dict(dims=(16, 16, 16), workers_list=(1,), precisions=("f64",), variants=("gather", "redblack"), reps=3)
    ours = {(r.operation, r.variant): r.checksum for r in run_benchmark(**kw)}
    ref = {(r.operation, r.variant): r.checksum for r in rb.run_benchmark(**kw)}
    for key in [("apply_P", "-"), ("apply_Pt", "gather"), ("apply_Pt", "redblack"), ("ngf_value_grad", "gather")]:
        assert ours[key] == ref[key], key
