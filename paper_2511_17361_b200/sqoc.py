"""SQOC grid files — the output format of cmd_voxelize.

Layout (little-endian, packed):

    "SQOC"            4 bytes magic
    u32 version       1
    u32 nx, ny, nz
    f32 origin[3]
    f32 resolution
    u16 C             number of classes
    u8  labels[V]     x-fastest (index = x + nx*(y + ny*z)); 255 = free
    u8  has_vo        presence byte of the optional block
    f32 v_o[V]        only when has_vo == 1

Writes are atomic (temp file + rename) and byte-identical for
identical inputs (SPEC.md:635 acceptance #9).
"""
from __future__ import annotations

import os
import struct
import tempfile
from dataclasses import dataclass

import numpy as np

MAGIC = b"SQOC"
VERSION = 1
FREE = 255
_HDR = struct.Struct("<4sIIII3ffH")


@dataclass
class SqocGrid:
    dims: tuple            # (nx, ny, nz)
    origin: tuple          # float32-rounded on disk
    resolution: float
    n_classes: int
    labels: np.ndarray     # uint8, memory order x-fastest, shape (nz, ny, nx); 255 = free
    v_o: np.ndarray | None = None  # float32, same shape


def _x_fastest(a: np.ndarray, dims, logical: bool) -> np.ndarray:
    """x-fastest memory order (nz, ny, nx) of ``a``.

    ``logical=False``: ``a`` already is the memory-order array (nz, ny, nx)
    (or any array with that C-order element sequence).  ``logical=True``: ``a``
    is the SPEC's logical (nx, ny, nz) view (``SemanticGrid.labels``,
    ``DenseGrids.v_o``) and is transposed.  The layout is never inferred from
    the shape: for nx == nz both layouts have the same shape."""
    nx, ny, nz = dims
    if logical:
        if a.shape != (nx, ny, nz):
            raise ValueError(f"logical grid must have shape {(nx, ny, nz)}, got {a.shape}")
        a = a.transpose(2, 1, 0)
    elif a.size != nx * ny * nz:
        raise ValueError(f"grid has {a.size} voxels, dims {(nx, ny, nz)} need {nx * ny * nz}")
    return np.ascontiguousarray(a.reshape(nz, ny, nx))


def write(path: str, dims, origin, resolution: float, n_classes: int, labels,
          free_index: int | None = None, v_o=None, *, logical: bool = False) -> None:
    """Write a grid.  ``labels`` uses ``free_index`` (default C) for free
    voxels; it is stored as 255.  ``labels`` / ``v_o`` are memory-order
    (nz, ny, nx) arrays, or logical (nx, ny, nz) views with ``logical=True``."""
    nx, ny, nz = (int(d) for d in dims)
    if n_classes < 1 or n_classes > 255:
        raise ValueError("SQOC stores 1..255 classes")
    free = n_classes if free_index is None else int(free_index)
    lab = _x_fastest(np.asarray(labels), (nx, ny, nz), logical).astype(np.int64)
    if np.any(((lab < 0) | (lab >= n_classes)) & (lab != free)):
        raise ValueError("labels outside [0, C) that are not the free index")
    lab = np.where(lab == free, FREE, lab).astype(np.uint8)
    hdr = _HDR.pack(MAGIC, VERSION, nx, ny, nz, *(float(o) for o in origin), float(resolution),
                    int(n_classes))
    body = [hdr, lab.tobytes()]
    if v_o is None:
        body.append(b"\x00")
    else:
        vo = _x_fastest(np.asarray(v_o, dtype=np.float32), (nx, ny, nz), logical).astype("<f4")
        body += [b"\x01", vo.tobytes()]
    d = os.path.dirname(os.path.abspath(path))
    fd, tmp = tempfile.mkstemp(dir=d, prefix=".sqoc.")
    try:
        with os.fdopen(fd, "wb") as fh:
            for b in body:
                fh.write(b)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def read(path: str) -> SqocGrid:
    with open(path, "rb") as fh:
        data = fh.read()
    if len(data) < _HDR.size or data[:4] != MAGIC:
        raise ValueError("not an SQOC file")
    magic, ver, nx, ny, nz, ox, oy, oz, res, C = _HDR.unpack_from(data, 0)
    if ver != VERSION:
        raise ValueError(f"unsupported SQOC version {ver}")
    V = nx * ny * nz
    o = _HDR.size
    if len(data) < o + V + 1:
        raise ValueError("truncated SQOC file")
    labels = np.frombuffer(data, np.uint8, V, o).reshape(nz, ny, nx).copy()
    o += V
    has_vo = data[o]
    o += 1
    v_o = None
    if has_vo == 1:
        if len(data) != o + 4 * V:
            raise ValueError("truncated SQOC v_o block")
        v_o = np.frombuffer(data, "<f4", V, o).reshape(nz, ny, nx).astype(np.float32)
    elif has_vo != 0 or len(data) != o:
        raise ValueError("malformed SQOC trailer")
    return SqocGrid((nx, ny, nz), (ox, oy, oz), res, C, labels, v_o)


def write_semantic_grid(path: str, sem, dense=None) -> None:
    """Write a SemanticGrid (+ optional DenseGrids.v_o) from voxelize(): both
    hold the SPEC's logical (nx, ny, nz) views."""
    write(path, sem.spec.dims, sem.spec.origin, sem.spec.resolution, len(sem.classes),
          sem.labels, sem.classes.free_index, None if dense is None else dense.v_o,
          logical=True)
