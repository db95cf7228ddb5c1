"""Frame-stack host side (PGM parsing/writing, reference io.py:83-150): CPU only."""

import os

import numpy as np
import pytest

from paper_2206_13369_b200 import frames as F


def _split(g, key, sizes):
    blob = g[key].tobytes()
    out, o = [], 0
    for n in g[sizes]:
        out.append(blob[o:o + int(n)])
        o += int(n)
    return out


def test_read_pgm_golden(golden, tmp_path):
    g = golden("frames")
    for j, data in enumerate(_split(g, "files", "file_sizes")):
        p = tmp_path / f"f{j}.pgm"
        p.write_bytes(data)
        assert np.array_equal(F.read_pgm(str(p)), g["raster"][j])  # incl. the commented header


def test_write_pgm_canonical(golden, tmp_path):
    g = golden("frames")
    files = _split(g, "files", "file_sizes")
    p = tmp_path / "x.pgm"
    F.write_pgm(g["raster"][0], str(p))
    assert p.read_bytes() == files[0]  # frame 0 was written by the reference's write_pgm
    with pytest.raises(ValueError):
        F.write_pgm(np.zeros(4, np.uint8), str(p))


def test_pgm_errors(tmp_path):
    bad = {
        "p2.pgm": b"P2\n2 2\n255\n0 0 0 0\n",
        "deep.pgm": b"P5\n2 2\n65535\n" + bytes(8),
        "short.pgm": b"P5\n4 4\n255\n" + bytes(5),
        "nohdr.pgm": b"P5\n4",
    }
    for name, data in bad.items():
        p = tmp_path / name
        p.write_bytes(data)
        with pytest.raises(F.FormatError):
            F.read_pgm(str(p))


def test_read_frames_validation(tmp_path):
    a, b = tmp_path / "a.pgm", tmp_path / "b.pgm"
    F.write_pgm(np.zeros((3, 4), np.uint8), str(a))
    F.write_pgm(np.zeros((4, 3), np.uint8), str(b))
    with pytest.raises(ValueError, match="no frames"):
        F.read_frames([])
    with pytest.raises(ValueError, match="expected 3x4"):
        F.read_frames([str(a), str(b)])
    r = F.read_frames([str(a), str(a)])
    assert r.shape == (2, 3, 4) and r.dtype == np.uint8
    assert not os.path.exists(tmp_path / "out")
