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
    sqoc.write(str(p), dims, (0, 0, 0), 1.0, 3, logical, free_index=200, logical=True)
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


@pytest.mark.parametrize("dims", [(3, 2, 3), (4, 4, 4), (5, 3, 5)])
def test_nx_equal_nz_logical_and_memory_order(tmp_path, dims):
    """nx == nz: the logical (nx, ny, nz) view and the memory-order
    (nz, ny, nx) array share a shape, so the layout is explicit, never
    inferred.  Both spellings of the same grid give the same file."""
    nx, ny, nz = dims
    rng = np.random.default_rng(sum(dims))
    mem = rng.integers(0, 6, size=(nz, ny, nx))          # free = 5 = C
    vo = rng.random((nz, ny, nx)).astype(np.float32)
    logical, vo_l = mem.transpose(2, 1, 0), vo.transpose(2, 1, 0)
    p1, p2 = tmp_path / "m.sqoc", tmp_path / "l.sqoc"
    sqoc.write(str(p1), dims, (0, 0, 0), 0.5, 5, mem, v_o=vo)
    sqoc.write(str(p2), dims, (0, 0, 0), 0.5, 5, logical, v_o=vo_l, logical=True)
    assert p1.read_bytes() == p2.read_bytes()
    g = sqoc.read(str(p1))
    np.testing.assert_array_equal(g.labels, np.where(mem == 5, 255, mem))
    np.testing.assert_array_equal(g.v_o, vo)
    # the on-disk index is x + nx*(y + ny*z)
    x, y, z = nx - 1, 0, 1
    raw = np.frombuffer(p1.read_bytes(), np.uint8, nx * ny * nz, sqoc._HDR.size)
    assert raw[x + nx * (y + ny * z)] == (255 if mem[z, y, x] == 5 else mem[z, y, x])


def test_write_semantic_grid_cubic_roundtrip(tmp_path):
    """write_semantic_grid on a grid with nx == nz (the SPEC's 32^3 example
    shape class): the labels read back equal the memory-order labels."""
    from paper_2511_17361_b200.core import ClassTable
    from paper_2511_17361_b200.voxelize import DenseGrids, SemanticGrid, VoxelGridSpec
    spec = VoxelGridSpec((0.0, 0.0, 0.0), (6, 4, 6), 0.5)
    rng = np.random.default_rng(3)
    mem = rng.integers(0, 4, size=(6, 4, 6))              # (nz, ny, nx); free = 3
    vo = rng.random((6, 4, 6)).astype(np.float32)
    sem = SemanticGrid(mem.transpose(2, 1, 0), spec, ClassTable(("a", "b", "c")))
    dense = DenseGrids(vo.transpose(2, 1, 0), None)
    p = tmp_path / "s.sqoc"
    sqoc.write_semantic_grid(str(p), sem, dense)
    g = sqoc.read(str(p))
    np.testing.assert_array_equal(g.labels, np.where(mem == 3, 255, mem))
    np.testing.assert_array_equal(g.v_o, vo)


def test_layout_mismatch_rejected(tmp_path):
    with pytest.raises(ValueError):
        sqoc.write(str(tmp_path / "x"), (4, 3, 2), (0, 0, 0), 1.0, 3, np.zeros((2, 3, 4)),
                   logical=True)
    with pytest.raises(ValueError):
        sqoc.write(str(tmp_path / "y"), (4, 3, 2), (0, 0, 0), 1.0, 3, np.zeros(23))
