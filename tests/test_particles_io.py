"""Particle files (cli.py:57-112) through the native reader
and writer in libesp_b200.so (csrc/esp_io.cu).  Host code: runs without a
GPU.  Fixtures were written and read back by the reference
(tests/golden/make_golden.py particles)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, golden


@pytest.mark.parametrize("name", ["particles_ortho", "particles_tri"])
def test_read_matches_reference(name):
    from paper_2601_00161_b200 import read_particles
    g = golden(name)
    s = read_particles(os.path.join(GOLDEN, name + ".txt"))
    np.testing.assert_array_equal(s.cell.h, g["h"])
    np.testing.assert_array_equal(s.positions, g["pos"])
    np.testing.assert_array_equal(s.charges, g["q"])
    np.testing.assert_array_equal(s.masses, g["m"])


@pytest.mark.parametrize("name", ["particles_ortho", "particles_tri"])
def test_write_byte_identical_to_reference(name, tmp_path):
    """read -> write of the reference's file gives the reference's own
    read -> write output byte for byte."""
    from paper_2601_00161_b200 import read_particles, write_particles
    out = tmp_path / "w.txt"
    write_particles(out, read_particles(os.path.join(GOLDEN, name + ".txt")))
    assert out.read_bytes() == open(os.path.join(GOLDEN, name + "_2.txt"), "rb").read()


def test_round_trip_fixed_point(tmp_path):
    from paper_2601_00161_b200 import Cell, ParticleSystem, read_particles, write_particles
    rng = np.random.default_rng(0)
    s = ParticleSystem(cell=Cell.orthorhombic([5.0, 6.0, 7.0]),
                       positions=rng.uniform(0, 5, (6, 3)), charges=rng.standard_normal(6),
                       masses=rng.uniform(0.5, 2.0, 6))
    a, b, c = (tmp_path / k for k in ("a.txt", "b.txt", "c.txt"))
    write_particles(a, s)
    back = read_particles(a)
    np.testing.assert_allclose(back.positions, s.positions, rtol=0, atol=1e-14)
    np.testing.assert_array_equal(back.charges, s.charges)
    write_particles(b, back)
    write_particles(c, read_particles(b))
    assert b.read_bytes() == c.read_bytes()


def test_comments_blanks_and_diagnostics(tmp_path):
    from paper_2601_00161_b200 import InputError, read_particles
    p = tmp_path / "c.txt"
    p.write_text("# header comment\n\ncell 5 5 5\n1 2 3 1.0 1.0  # inline comment\n")
    assert read_particles(p).n == 1
    bad = tmp_path / "bad.txt"
    bad.write_text("cell 5 5 5\n1 2 oops 1.0 1.0\n")
    with pytest.raises(InputError, match=r"bad\.txt:2:3"):
        read_particles(bad)
    nohdr = tmp_path / "nohdr.txt"
    nohdr.write_text("1 2 3 1.0 1.0\n")
    with pytest.raises(InputError, match="header"):
        read_particles(nohdr)
    cols = tmp_path / "cols.txt"
    cols.write_text("cell 5 5 5\n1 2 3 1.0\n")
    with pytest.raises(InputError, match="5 columns"):
        read_particles(cols)
    empty = tmp_path / "empty.txt"
    empty.write_text("cell 5 5 5\n")
    with pytest.raises(InputError, match="no particle lines"):
        read_particles(empty)
    hdr = tmp_path / "hdr.txt"
    hdr.write_text("cell3 1 2 3\n")
    with pytest.raises(InputError, match="9 entries"):
        read_particles(hdr)
    neg = tmp_path / "neg.txt"
    neg.write_text("cell 5 5 5\n1 2 3 1.0 -1.0\n")
    with pytest.raises(InputError, match="masses"):
        read_particles(neg)
    with pytest.raises(InputError):
        read_particles(tmp_path / "missing.txt")


def _python_rows(path):
    """The reference reader's line and token rules (cli.py:57-88), applied
    with Python's own str.splitlines / str.split / float."""
    from pathlib import Path
    hdr, rows = None, []
    for ln, raw in enumerate(Path(path).read_text().splitlines(), start=1):
        text = raw.split("#", 1)[0].strip()
        if not text:
            continue
        cols = text.split()
        if hdr is None:
            hdr = [float(c) for c in cols[1:]]
            continue
        rows.append([float(c) for c in cols] + [ln])
    return hdr, rows


@pytest.mark.parametrize("body", [
    "cell 5 5 6\r1 2 3 0.5 1\r4 1_0e-1 2 -0.5 2\r",              # CR-only lines, underscore
    "cell 5 5 6\r\n1 2 3 0.5 1\r\n\r\n4 1 2 -0.5 2",              # CRLF, blank, no final EOL
    "cell 5 5 6\x0b1 2 3 0.5 1\x0c4 1 2 -0.5 2\x1c3 3 3 1 1\n",   # \v \f \x1c line breaks
    "cell 5 5 6 1 2 3 0.5 1  4 1 2 -0.5 2\x85",    # U+2028/2029/0085, NBSP
    "cell\x1f5 5 6\n1　2 3 0.5 1\n1_000e-3 2 3 0.5 1\n",      # \x1f and U+3000 separators
])
def test_line_breaks_and_tokens_follow_python(tmp_path, body):
    from paper_2601_00161_b200 import read_particles
    p = tmp_path / "p.txt"
    p.write_bytes(body.encode("utf-8"))
    hdr, rows = _python_rows(p)
    s = read_particles(p)
    np.testing.assert_array_equal(np.diag(s.cell.h), hdr)
    want = np.array([r[:5] for r in rows])
    np.testing.assert_array_equal(s.positions, s.cell.wrap(want[:, :3]))
    np.testing.assert_array_equal(s.charges, want[:, 3])


@pytest.mark.parametrize("tok", ["1__0", "_1", "1_", "1._5", "nan(1)", "0x10"])
def test_tokens_python_float_rejects(tmp_path, tok):
    from paper_2601_00161_b200 import InputError, read_particles
    with pytest.raises(ValueError):
        float(tok)
    p = tmp_path / "t.txt"
    p.write_text(f"cell 5 5 5\n1 2 3 {tok} 1\n")
    with pytest.raises(InputError, match=r"t\.txt:2:4"):
        read_particles(p)


def test_cr_only_diagnostic_line_numbers(tmp_path):
    from paper_2601_00161_b200 import InputError, read_particles
    p = tmp_path / "cr.txt"
    p.write_bytes(b"cell 5 5 5\r1 2 3 1 1\r1 2 x 1 1\r")
    with pytest.raises(InputError, match=r"cr\.txt:3:3"):
        read_particles(p)
