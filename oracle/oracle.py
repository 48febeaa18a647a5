"""ctypes binding of oracle/sqv_oracle.c — TEST INFRASTRUCTURE ONLY.

The oracle is the parity checker and CPU baseline of the B200 voxelizer.  It
restates the reference's per-point math (/root/reference/pkg/src/sqocc/
core.py:30-35,55-65,143-173,237-282) and the SPEC voxelize glue
 in plain C / FP64; see the header
of sqv_oracle.c for the line-by-line map.  It is pinned against golden vectors
produced by the reference's own ``sqocc.core`` (tests/golden/make_golden.py).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline, --impl
reference) may import this module.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libsqv_oracle.so")
_lib = None

TILE = (8, 8, 16)  # SQV_TILE_X/Y/Z of include/sqv.h


def build(force: bool = False) -> str:
    """Compile the oracle with oracle/Makefile (gcc, OpenMP)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(
            os.path.join(_HERE, "sqv_oracle.c")):
        subprocess.run(["make", "-C", _HERE, "-B" if force else "all"], check=True,
                       stdout=subprocess.DEVNULL)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        i32, i64, f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        L.sqvo_prep.argtypes = [i32, i32, i32, P, P, P, P, P, P, P, P, P, f64, f64, i32, i32,
                                i32, i32, f64, P, P, P]
        L.sqvo_bins.argtypes = [i32, i32, P, P, P, P, i64, P]
        L.sqvo_voxelize.argtypes = [i32, i32, i32, P, P, P, P, P, P, P, P, P, f64, f64, i32, i32,
                                    i32, i32, f64, P, P, P, P, P, P]
        L.sqvo_finalize.argtypes = [P, P, i64, i32, f64, i32, P]
        L.sqvo_finalize.restype = None
        L.sqvo_confusion.argtypes = [P, P, i64, i32, P]
        L.sqvo_confusion.restype = None
        L.sqvo_density.argtypes = [i32, i32, P, P, P, P, P, P, P, P, i64, P, P]
        L.sqvo_set_threads.argtypes = [i32]
        L.sqvo_set_threads.restype = None
        L.sqvo_ray_iou.argtypes = [i32, P, P, P, P, f64, i32, i64, P, P, i32, P, P, P, P, P, P]
        L.sqvo_ray_iou.restype = None
        _lib = L
    return _lib


def threads() -> int:
    return int(lib().sqvo_threads())


def set_threads(n: int) -> None:
    lib().sqvo_set_threads(int(n))


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class Prims:
    """FP64 SoA inputs, frame-major (same layout as include/sqv.h sqv_prims)."""
    mu: np.ndarray       # [F,N,3]
    scale: np.ndarray    # [F,N,3]
    rot: np.ndarray      # [F,N,4] (w,x,y,z)
    opacity: np.ndarray  # [F,N]
    eps: np.ndarray      # [F,N,2] (eps1, eps2)
    logits: np.ndarray   # [F,N,C]
    n_valid: np.ndarray | None = None  # [F] int32

    @staticmethod
    def of(obj) -> "Prims":
        f = lambda a: np.ascontiguousarray(np.asarray(a), dtype=np.float64)
        nv = getattr(obj, "n_valid", None)
        if nv is not None:
            nv = np.ascontiguousarray(np.asarray(nv), dtype=np.int32)
        p = Prims(f(obj.mu), f(obj.scale), f(obj.rot), f(obj.opacity), f(obj.eps),
                  f(obj.logits), nv)
        if p.mu.ndim == 2:  # single frame
            p = Prims(p.mu[None], p.scale[None], p.rot[None], p.opacity[None], p.eps[None],
                      p.logits[None], nv)
        return p

    @property
    def shape(self):
        F, N = self.opacity.shape
        return F, N, self.logits.shape[2]


@dataclass
class Grid:
    origin: tuple = (-40.0, -40.0, -1.0)
    dims: tuple = (200, 200, 16)
    resolution: float = 0.4


@dataclass
class Cfg:
    tau: float = 0.01
    neighborhood_radius: int = 5
    truncate: bool = True
    prob_sum: bool = False
    free_label: int = 255
    window_extent: float = 2.5


class InvalidPrimitive(ValueError):
    def __init__(self, index, bits):
        super().__init__(f"invalid primitive {index} (bits {bits})")
        self.index, self.bits = index, bits


def _common(p: Prims, g: Grid, c: Cfg):
    F, N, C = p.shape
    origin = np.asarray(g.origin, np.float64)
    dims = np.asarray(g.dims, np.int32)
    return (F, N, C, _p(p.mu), _p(p.scale), _p(p.rot), _p(p.opacity), _p(p.eps), _p(p.logits),
            _p(p.n_valid), _p(origin), _p(dims), float(g.resolution), float(c.tau),
            int(c.neighborhood_radius), int(bool(c.truncate)), int(bool(c.prob_sum)),
            int(c.free_label), float(c.window_extent)), (origin, dims)


def prep(p: Prims, g: Grid = Grid(), c: Cfg = Cfg()) -> np.ndarray:
    """Windows [F,N,6] (lo xyz, hi xyz; empty: lo > hi).  Raises InvalidPrimitive."""
    args, keep = _common(p, g, c)
    F, N, _ = p.shape
    win = np.zeros((F, N, 6), np.int32)
    bad = np.zeros(1, np.int64)
    bits = np.zeros(1, np.int32)
    rc = lib().sqvo_prep(*args, _p(win), _p(bad), _p(bits))
    if rc:
        raise InvalidPrimitive(int(bad[0]), int(bits[0]))
    return win


def bins(windows: np.ndarray, dims) -> tuple[np.ndarray, np.ndarray]:
    """(tile_off [F*T+1], prim_ids [entries]) — ascending primitive ids per tile."""
    windows = np.ascontiguousarray(windows, np.int32)
    F, N, _ = windows.shape
    dims = np.asarray(dims, np.int32)
    T = int(np.prod([(d + t - 1) // t for d, t in zip(dims, TILE)]))
    tile_off = np.zeros(F * T + 1, np.int32)
    n = np.zeros(1, np.int64)
    rc = lib().sqvo_bins(F, N, _p(windows), _p(dims), _p(tile_off), None, 0, _p(n))
    ids = np.zeros(max(int(n[0]), 1), np.int32)
    rc = lib().sqvo_bins(F, N, _p(windows), _p(dims), _p(tile_off), _p(ids), ids.size, _p(n))
    assert rc == 0
    return tile_off, ids[: int(n[0])]


def voxelize(p: Prims, g: Grid = Grid(), c: Cfg = Cfg(), want_vc: bool = True):
    """FP64 voxelize (+finalize).  Returns dict v_o [F,V], v_c [F,V,C] (or None),
    labels [F,V] u8, n_pairs.  Voxel index = x + nx*(y + ny*z)."""
    args, keep = _common(p, g, c)
    F, N, C = p.shape
    V = int(np.prod(g.dims))
    v_o = np.zeros((F, V), np.float64)
    v_c = np.zeros((F, V, C), np.float64) if want_vc else None
    labels = np.zeros((F, V), np.uint8)
    n_pairs = np.zeros(1, np.int64)
    bad = np.zeros(1, np.int64)
    bits = np.zeros(1, np.int32)
    rc = lib().sqvo_voxelize(*args, _p(v_o), _p(v_c), _p(labels), _p(n_pairs), _p(bad), _p(bits))
    if rc:
        raise InvalidPrimitive(int(bad[0]), int(bits[0]))
    return {"v_o": v_o, "v_c": v_c, "labels": labels, "n_pairs": int(n_pairs[0])}


def finalize(v_o, v_c, tau, free_label=255):
    v_o = np.ascontiguousarray(v_o, np.float64)
    v_c = np.ascontiguousarray(v_c, np.float64)
    n = v_o.size
    C = v_c.size // max(n, 1)
    out = np.zeros(n, np.uint8)
    lib().sqvo_finalize(_p(v_o), _p(v_c), n, C, float(tau), int(free_label), _p(out))
    return out.reshape(v_o.shape)


def confusion(pred, gt, n_classes):
    pred = np.ascontiguousarray(pred, np.uint8).ravel()
    gt = np.ascontiguousarray(gt, np.uint8).ravel()
    cm = np.zeros((n_classes + 1) * (n_classes + 1), np.int64)
    lib().sqvo_confusion(_p(pred), _p(gt), pred.size, int(n_classes), _p(cm))
    return cm.reshape(n_classes + 1, n_classes + 1)


def density(p: Prims, points, pair_prim):
    """(F, density) FP64 of primitive pair_prim[k] at world point points[k] (1 frame)."""
    F_, N, C = p.shape
    assert F_ == 1
    points = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
    pair_prim = np.ascontiguousarray(pair_prim, np.int32).ravel()
    n = points.shape[0]
    Fv = np.zeros(n, np.float64)
    dv = np.zeros(n, np.float64)
    rc = lib().sqvo_density(N, C, _p(p.mu), _p(p.scale), _p(p.rot), _p(p.opacity), _p(p.eps),
                            _p(p.logits), _p(points), _p(pair_prim), n, _p(Fv), _p(dv))
    if rc:
        raise InvalidPrimitive(-1, rc)
    return Fv, dv


def ray_iou(pred, gt, dims, origin, resolution, n_classes, origins, dirs, thresholds):
    """ray_iou counts.  pred/gt: [F][V] (or [V]) u8 labels,
    x-fastest; origins/dirs [R,3].  Returns (counts [T,3] int64 TP/FP/FN,
    hits dict of per-ray d/class arrays [F,R], class -1 = no hit)."""
    pred = np.ascontiguousarray(pred, np.uint8)
    gt = np.ascontiguousarray(gt, np.uint8)
    V = int(np.prod(dims))
    F = pred.size // V
    origins = np.ascontiguousarray(origins, np.float64).reshape(-1, 3)
    dirs = np.ascontiguousarray(dirs, np.float64).reshape(-1, 3)
    thr = np.ascontiguousarray(thresholds, np.float64).ravel()
    R = origins.shape[0]
    counts = np.zeros((thr.size, 3), np.int64)
    dp = np.zeros((F, R)); dg = np.zeros((F, R))
    cp = np.zeros((F, R), np.int32); cg = np.zeros((F, R), np.int32)
    d = np.ascontiguousarray(dims, np.int32)
    o = np.ascontiguousarray(origin, np.float64)
    lib().sqvo_ray_iou(F, _p(pred), _p(gt), _p(d), _p(o), float(resolution),
                       int(n_classes), R, _p(origins), _p(dirs), int(thr.size),
                       _p(thr), _p(counts), _p(dp), _p(cp), _p(dg), _p(cg))
    return counts, {"d_pred": dp, "c_pred": cp, "d_gt": dg, "c_gt": cg}
