"""MetaImage / landmark I/O (fileio.py:1-204) and the CLI's host-side contract
(cli.py:1-268: usage, I/O and grid errors, exit codes) -- no GPU needed.  The
reference-written files in tests/golden/ pin the byte format."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, grid_from, load_golden

import paper_1812_06765_b200 as ngf
from oracle import ngf_oracle as O
from paper_1812_06765_b200 import fileio
from paper_1812_06765_b200.cli import EXIT_IO, EXIT_NUMERIC, EXIT_USAGE, main


def _rewrite_identical(src, tmp_path, reader, writer):
    obj = reader(src)
    dst = str(tmp_path / os.path.basename(src))
    writer(obj, dst)
    assert open(dst, "rb").read() == open(src, "rb").read()
    return obj


def test_reference_written_files_read_and_rewrite_byte_identical(tmp_path):
    vol = _rewrite_identical(os.path.join(GOLDEN, "fio_vol_f32.mha"), tmp_path, fileio.read_volume,
                             fileio.write_volume)
    assert vol.grid == ngf.Grid3((6, 5, 4), (0.7, 1.25, 2.5), (-1.5, 0.25, 3.0))
    assert vol.values.dtype == np.float32 and vol.values.shape == (4, 5, 6)
    d = _rewrite_identical(os.path.join(GOLDEN, "fio_def_f64.mha"), tmp_path, fileio.read_deformation,
                           fileio.write_deformation)
    assert d.grid == ngf.Grid3((4, 3, 5), (2.0, 1.5, 2.5), (1.0, -2.0, 0.0))
    assert d.field.dtype == np.float64 and d.field.shape == (3, 5, 3, 4)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_volume_and_deformation_roundtrip(tmp_path, dtype):
    g = ngf.Grid3((5, 4, 3), (0.7, 1.25, 2.5), (-1.5, 0.25, 3.0))
    vals = np.random.default_rng(0).standard_normal(g.shape).astype(dtype)
    fileio.write_volume(ngf.Image3(g, vals), str(tmp_path / "v.mha"))
    back = fileio.read_volume(str(tmp_path / "v.mha"))
    assert back.grid == g and back.values.dtype == dtype and np.array_equal(back.values, vals)
    y = ngf.smooth_random_field(g, seed=3, amplitude_mm=1.5)
    y.field = y.field.astype(dtype)
    fileio.write_deformation(y, str(tmp_path / "y.mha"))
    yb = fileio.read_deformation(str(tmp_path / "y.mha"))
    assert yb.grid == g and np.array_equal(yb.field, y.field)


def test_int16_payload_is_promoted(tmp_path):
    g = ngf.Grid3((3, 3, 3), (1, 1, 1), (0, 0, 0))
    vals = (np.arange(27, dtype=np.int16) - 13).reshape(g.shape)
    fileio._write_meta(str(tmp_path / "ct.mha"), g, vals[..., None], channels=1)
    assert fileio.read_volume(str(tmp_path / "ct.mha")).values.dtype == np.float64
    back = fileio.read_volume(str(tmp_path / "ct.mha"), promote_dtype=np.float32)
    assert back.values.dtype == np.float32 and np.array_equal(back.values, vals.astype(np.float32))


def test_mhd_with_external_raw(tmp_path):
    vals = np.arange(12, dtype="<f8").reshape(2, 2, 3)
    (tmp_path / "v.raw").write_bytes(vals.tobytes())
    (tmp_path / "v.mhd").write_text("ObjectType = Image\nNDims = 3\nBinaryData = True\nDimSize = 3 2 2\n"
                                    "ElementType = MET_DOUBLE\nElementDataFile = v.raw\n")
    assert np.array_equal(fileio.read_volume(str(tmp_path / "v.mhd")).values, vals)


def test_malformed_files_raise_metaimage_error(tmp_path):
    g = ngf.Grid3((4, 4, 4), (1, 1, 1), (0, 0, 0))
    p = str(tmp_path / "t.mha")
    fileio.write_volume(ngf.smooth_random_volume(g, seed=2), p)
    data = open(p, "rb").read()
    open(p, "wb").write(data[:-16])
    with pytest.raises(fileio.MetaImageError, match="truncated"):
        fileio.read_volume(p)
    bad = tmp_path / "bad.mha"
    for text, msg in [("ObjectType = Image\nNDims = 2\nElementDataFile = LOCAL\n", "NDims"),
                      ("NDims = 3\nDimSize = 1 1 1\nElementType = MET_UCHAR\nElementDataFile = LOCAL\n",
                       "ElementType"),
                      ("no equals sign here\n", "malformed"),
                      ("NDims = 3\nDimSize = 2 2 2\nElementType = MET_FLOAT\nCompressedData = True\n"
                       "ElementDataFile = LOCAL\n", "ompressed"),
                      ("NDims = 3\nDimSize = 2 2\nElementType = MET_FLOAT\nElementDataFile = LOCAL\n", "3 entries")]:
        bad.write_text(text)
        with pytest.raises(fileio.MetaImageError, match=msg):
            fileio.read_volume(str(bad))
    with pytest.raises(fileio.MetaImageError):
        fileio.read_volume(str(tmp_path / "missing.mha"))
    assert issubclass(fileio.MetaImageError, ValueError) and issubclass(fileio.LandmarkFileError, ValueError)


def test_channel_checks(tmp_path):
    g = ngf.Grid3((3, 3, 3), (1, 1, 1), (0, 0, 0))
    fileio.write_volume(ngf.smooth_random_volume(g, seed=4), str(tmp_path / "v.mha"))
    fileio.write_deformation(ngf.make_identity(g), str(tmp_path / "d.mha"))
    with pytest.raises(fileio.MetaImageError, match="channels"):
        fileio.read_volume(str(tmp_path / "d.mha"))
    with pytest.raises(fileio.MetaImageError, match="channels"):
        fileio.read_deformation(str(tmp_path / "v.mha"))


def test_landmark_frames_and_errors(tmp_path):
    g = ngf.Grid3((10, 10, 10), (0.97, 0.97, 2.5), (0.0, 0.0, 0.0))
    p = tmp_path / "lm.txt"
    p.write_text("1 1 1\n3 2 5\n\n")
    lm = fileio.read_landmarks(str(p), "index1", g)  # DIR-lab 1-based convention
    assert lm.count == 2 and np.allclose(lm.points[1], [2 * 0.97, 0.97, 4 * 2.5])
    g2 = ngf.Grid3((5, 5, 5), (2.0, 2.0, 2.0), (1.0, 1.0, 1.0))
    p.write_text("1 2 3\n")
    assert np.allclose(fileio.read_landmarks(str(p), "index0", g2).points[0], [3.0, 5.0, 7.0])
    assert np.allclose(fileio.read_landmarks(str(p), "world", g2).points[0], [1.0, 2.0, 3.0])
    with pytest.raises(ValueError):
        fileio.read_landmarks(str(p), "voxels", g2)
    p.write_text("1 2\n")
    with pytest.raises(fileio.LandmarkFileError, match="expected 3"):
        fileio.read_landmarks(str(p), "world", g2)
    p.write_text("1 2 x\n")
    with pytest.raises(fileio.LandmarkFileError, match="non-numeric"):
        fileio.read_landmarks(str(p), "world", g2)


def test_oracle_sample_deformation_matches_reference_fixture():
    z = load_golden("evaluation")
    for k in range(int(z["n"])):
        g = grid_from(z[f"{k}_g"])
        assert np.array_equal(O.sample_deformation(z[f"{k}_y"], g, z[f"{k}_pts"]), z[f"{k}_sample"])


def test_cli_usage_and_io_errors(tmp_path):
    assert main([]) == EXIT_USAGE
    assert main(["register"]) == EXIT_USAGE
    assert main(["register", "--reference", "a"]) == EXIT_USAGE
    assert main(["frobnicate"]) == EXIT_USAGE
    assert main(["benchmark", "--dims", "12,12"]) == EXIT_USAGE
    assert main(["register", "--reference", str(tmp_path / "no.mha"), "--template", str(tmp_path / "no2.mha"),
                 "--out-deformation", str(tmp_path / "y.mha")]) == EXIT_IO


def test_cli_grid_mismatch_is_numeric_error_with_hint(tmp_path, capsys):
    a, b = str(tmp_path / "a.mha"), str(tmp_path / "b.mha")
    fileio.write_volume(ngf.smooth_random_volume(ngf.Grid3((8, 8, 8), (1, 1, 1), (0, 0, 0)), seed=1), a)
    fileio.write_volume(ngf.smooth_random_volume(ngf.Grid3((8, 8, 8), (1.5, 1, 1), (0, 0, 0)), seed=2), b)
    assert main(["register", "--reference", a, "--template", b, "--out-deformation",
                 str(tmp_path / "y.mha")]) == EXIT_NUMERIC
    assert "resample" in capsys.readouterr().err


def test_cli_warp_difference_needs_reference_and_bad_landmarks_are_io_errors(tmp_path):
    g = ngf.Grid3((8, 8, 8), (2, 2, 2), (0, 0, 0))
    tp, yp, lm = str(tmp_path / "t.mha"), str(tmp_path / "y.mha"), str(tmp_path / "lm.txt")
    fileio.write_volume(ngf.smooth_random_volume(g, seed=1), tp)
    fileio.write_deformation(ngf.make_identity(ngf.deformation_grid_for(g, 4)), yp)
    assert main(["warp", "--template", tp, "--deformation", yp, "--out", str(tmp_path / "w.mha"),
                 "--out-difference", str(tmp_path / "d.mha")]) == EXIT_USAGE
    open(lm, "w").write("1 2\n")
    assert main(["evaluate", "--deformation", yp, "--landmarks-ref", lm, "--landmarks-template", lm,
                 "--image-grid-from", tp, "--frame", "index1"]) == EXIT_IO
