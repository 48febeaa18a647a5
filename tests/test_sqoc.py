"""SQOC grid format: write->read bit-exact, byte-identical repeats."""
import os

import numpy as np
import pytest

from paper_2511_17361_b200 import sqoc


def test_roundtrip_bit_exact_and_byte_identical(tmp_path):
    rng = np.random.default_rng(1)
    dims = (7, 5, 3)
    C = 4
    lab = rng.integers(0, C + 1, size=(3, 5, 7))          # memory order, free = C
    vo = rng.random((3, 5, 7)).astype(np.float32)
    p1, p2 = tmp_path / "a.sqoc", tmp_path / "b.sqoc"
    sqoc.write(str(p1), dims, (-1.5, 2.0, 0.25), 0.4, C, lab, v_o=vo)
    sqoc.write(str(p2), dims, (-1.5, 2.0, 0.25), 0.4, C, lab, v_o=vo)
    assert p1.read_bytes() == p2.read_bytes()
    g = sqoc.read(str(p1))
    assert g.dims == dims and g.n_classes == C
    np.testing.assert_array_equal(g.labels, np.where(lab == C, 255, lab))
    assert g.v_o.dtype == np.float32 and np.array_equal(g.v_o, vo)
    b = p1.read_bytes()
    assert b[:4] == b"SQOC" and int.from_bytes(b[4:8], "little") == 1
    assert len(b) == 4 + 4 * 4 + 4 * 4 + 2 + 105 + 1 + 4 * 105


def test_logical_view_and_no_vo(tmp_path):
    dims = (4, 3, 2)
    mem = np.arange(24).reshape(2, 3, 4) % 3            # (nz, ny, nx), classes 0..2
    logical = mem.transpose(2, 1, 0)                     # (nx, ny, nz) view
    p = tmp_path / "c.sqoc"
    sqoc.write(str(p), dims, (0, 0, 0), 1.0, 3, logical, free_index=200)
    g = sqoc.read(str(p))
    np.testing.assert_array_equal(g.labels, mem)
    assert g.v_o is None


def test_rejects_bad_input(tmp_path):
    with pytest.raises(ValueError):
        sqoc.write(str(tmp_path / "x"), (2, 1, 1), (0, 0, 0), 1.0, 2, np.array([0, 7]))
    bad = tmp_path / "bad.sqoc"
    bad.write_bytes(b"NOPE" + bytes(40))
    with pytest.raises(ValueError):
        sqoc.read(str(bad))
    assert not any(n.startswith(".sqoc.") for n in os.listdir(tmp_path))
