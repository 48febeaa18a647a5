"""Occupancy metrics of SPEC.md:481-546 over device confusion counts.

- ``confusion_matrix(pred, gt, n_classes)`` — K6 kernel (include/sqv.h
  ``sqv_confusion``): (C+1)x(C+1) int64 counts, row = gt, col = pred,
  index C = free.  Integer sums: bit-exact and order-independent.
- ``voxel_iou(pred, gt)``  SPEC.md:494-502 — binary occupied IoU; 1.0 if
  both grids are fully free.
- ``miou(pred, gt)``       SPEC.md:504-512 — per-class IoU (free excluded),
  classes absent from both grids excluded from the mean.
- ``iou_from_confusion`` / ``miou_from_confusion`` — the same folds over a
  count matrix (e.g. one all-reduced over ranks, see distributed.py).

- ``ray_iou(pred, gt, origins, dirs, thresholds)`` SPEC.md:514-523 — per ray
  the first occupied voxel of each grid by a 3D DDA (device kernel
  ``sqv_ray_iou``), TP/FP/FN per threshold as int64 counts, RayIoU@t =
  TP / (TP + FP + FN).  ``default_rays`` is the SPEC design-decision fan.
"""
from __future__ import annotations

import numpy as np

from . import _lib


def _device_u8(a, device):
    import torch
    if isinstance(a, torch.Tensor):
        return a.to(device=device).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a)).to(device)


def _labels_u8(grid_labels, C, free_index):
    """SemanticGrid labels (any int dtype, free = free_index) -> u8 with free -> 255."""
    a = np.asarray(grid_labels)
    if a.dtype == np.uint8 and (free_index >= C and free_index <= 255):
        return a
    a = a.astype(np.int64)
    return np.where((a >= 0) & (a < C), a, 255).astype(np.uint8)


def confusion_matrix(pred, gt, n_classes: int, out=None, stream=None):
    """(C+1)^2 int64 counts on the device.  pred/gt: uint8 label arrays or
    device tensors of equal size; labels >= C count as free.  Accumulates into
    ``out`` (a zeroed int64 device tensor) when given."""
    import torch
    dev = _lib.require_cuda()
    L = _lib.lib()
    p = _device_u8(pred, dev)
    g = _device_u8(gt, dev)
    if p.numel() != g.numel():
        raise ValueError("dimension mismatch")
    if not (1 <= n_classes <= 255):
        raise ValueError("n_classes must lie in [1, 255]")
    K = n_classes + 1
    if out is None:
        out = torch.zeros((K, K), dtype=torch.int64, device=dev)
    s = stream if stream is not None else _lib.stream_ptr(dev)
    _lib.check(L.sqv_confusion(p.data_ptr(), g.data_ptr(), p.numel(), n_classes, 255,
                               out.data_ptr(), s), "sqv_confusion")
    return out


def iou_from_confusion(cm) -> float:
    """Binary occupied/free IoU from (C+1)^2 counts."""
    cm = np.asarray(cm, dtype=np.int64)
    C = cm.shape[0] - 1
    inter = int(cm[:C, :C].sum())
    union = int(cm.sum() - cm[C, C])
    return 1.0 if union == 0 else inter / union


def miou_from_confusion(cm) -> tuple[np.ndarray, float, np.ndarray]:
    """(per-class IoU, mIoU, valid mask) from counts."""
    cm = np.asarray(cm, dtype=np.int64)
    C = cm.shape[0] - 1
    tp = np.diag(cm)[:C].astype(np.float64)
    union = cm[:C, :].sum(1) + cm[:, :C].sum(0) - np.diag(cm)[:C]
    valid = union > 0
    per = np.zeros(C)
    per[valid] = tp[valid] / union[valid]
    m = float(per[valid].mean()) if valid.any() else float("nan")
    return per, m, valid


def _check_pair(pred, gt):
    if tuple(pred.spec.dims) != tuple(gt.spec.dims):
        raise ValueError("dimension mismatch")
    if len(pred.classes) != len(gt.classes):
        raise ValueError("class tables differ")


def _grid_cm(pred, gt):
    _check_pair(pred, gt)
    C = len(pred.classes)
    # x-fastest memory order of the logical (nx, ny, nz) arrays is irrelevant to
    # counting, but pred and gt must be traversed identically: use the same view.
    p = _labels_u8(np.asarray(pred.labels).transpose(2, 1, 0), C, pred.classes.free_index)
    g = _labels_u8(np.asarray(gt.labels).transpose(2, 1, 0), C, gt.classes.free_index)
    return confusion_matrix(p, g, C).cpu().numpy()


def voxel_iou(pred, gt) -> float:
    return iou_from_confusion(_grid_cm(pred, gt))


def miou(pred, gt) -> tuple[np.ndarray, float]:
    per, m, _ = miou_from_confusion(_grid_cm(pred, gt))
    return per, m


# ---- RayIoU ------------------------------------------------

DEFAULT_THRESHOLDS = (1.0, 2.0, 4.0)
# SPEC.md "DESIGN DECISIONS": a horizontal fan from the grid centre, 360
# azimuths x 4 elevations (the elevations are this implementation's choice).
DEFAULT_ELEVATIONS_DEG = (-10.0, -5.0, 0.0, 5.0)


def default_rays(spec, n_azimuth: int = 360, elevations_deg=DEFAULT_ELEVATIONS_DEG,
                 origin=None) -> tuple[np.ndarray, np.ndarray]:
    """(origins [R,3], unit dirs [R,3]) FP64, R = n_azimuth x len(elevations):
    azimuth k * 360/n_azimuth degrees, elevation-major."""
    if n_azimuth < 1 or len(elevations_deg) < 1:
        raise ValueError("zero rays")
    if origin is None:
        origin = (np.asarray(spec.origin, np.float64)
                  + np.asarray(spec.dims, np.float64) * float(spec.resolution) / 2.0)
    az = np.arange(n_azimuth, dtype=np.float64) * (2.0 * np.pi / n_azimuth)
    el = np.deg2rad(np.asarray(elevations_deg, np.float64))
    E, A = np.meshgrid(el, az, indexing="ij")
    dirs = np.stack([np.cos(E) * np.cos(A), np.cos(E) * np.sin(A), np.sin(E)], -1).reshape(-1, 3)
    origins = np.broadcast_to(np.asarray(origin, np.float64), dirs.shape).copy()
    return origins, dirs


def _check_rays(origins, dirs):
    o = np.ascontiguousarray(origins, np.float64).reshape(-1, 3)
    d = np.ascontiguousarray(dirs, np.float64).reshape(-1, 3)
    if o.shape[0] == 0 or d.shape[0] == 0:
        raise ValueError("zero rays")
    if o.shape != d.shape:
        raise ValueError("origins and dirs must both be [R, 3]")
    if not (np.isfinite(o).all() and np.isfinite(d).all()):
        raise ValueError("origins and dirs must be finite")
    if np.abs(np.linalg.norm(d, axis=1) - 1.0).max() > 1e-6:
        raise ValueError("dirs must be unit 3-vectors")
    return o, d


def ray_counts(pred, gt, spec, n_classes: int, origins, dirs, thresholds=DEFAULT_THRESHOLDS,
               out=None, return_hits: bool = False, stream=None):
    """Device TP/FP/FN counts [T, 3] int64 of ray_iou over [F][V] (or [V])
    u8 label grids, x-fastest, labels >= n_classes free.  Accumulates into
    ``out`` when given.  With return_hits, also the per-ray hit distances
    (-1 = none) and classes (-1 = none), [F, R] each."""
    import torch
    o, d = _check_rays(origins, dirs)
    thr = np.ascontiguousarray(thresholds, np.float64).ravel()
    if thr.size < 1 or thr.size > 16 or not (thr >= 0).all():
        raise ValueError("1..16 thresholds, each >= 0")
    if not (1 <= n_classes <= 255):
        raise ValueError("n_classes must lie in [1, 255]")
    dev = _lib.require_cuda()
    L = _lib.lib()
    p = _device_u8(pred, dev)
    g = _device_u8(gt, dev)
    V = int(np.prod(spec.dims))
    if p.numel() != g.numel() or p.numel() % V:
        raise ValueError("dimension mismatch")
    F = p.numel() // V
    R = o.shape[0]
    od = torch.from_numpy(o).to(dev)
    dd = torch.from_numpy(d).to(dev)
    if out is None:
        out = torch.zeros((thr.size, 3), dtype=torch.int64, device=dev)
    hits = None
    hp = None
    if return_hits:
        hits = {"d_pred": torch.empty((F, R), dtype=torch.float64, device=dev),
                "c_pred": torch.empty((F, R), dtype=torch.int32, device=dev),
                "d_gt": torch.empty((F, R), dtype=torch.float64, device=dev),
                "c_gt": torch.empty((F, R), dtype=torch.int32, device=dev)}
        hp = _lib.RayHits(hits["d_pred"].data_ptr(), hits["c_pred"].data_ptr(),
                          hits["d_gt"].data_ptr(), hits["c_gt"].data_ptr())
    grid = spec._c()
    s = stream if stream is not None else _lib.stream_ptr(dev)
    import ctypes
    _lib.check(L.sqv_ray_iou(p.data_ptr(), g.data_ptr(), F, ctypes.byref(grid), n_classes,
                             od.data_ptr(), dd.data_ptr(), R, thr.ctypes.data, thr.size,
                             out.data_ptr(), ctypes.byref(hp) if hp is not None else None, s),
               "sqv_ray_iou")
    return (out, hits) if return_hits else out


def rayiou_from_counts(counts, thresholds=DEFAULT_THRESHOLDS) -> dict:
    """{threshold: TP / (TP + FP + FN)} from [T, 3] counts; 1.0 when no ray
    hits in either grid (both empty along every ray)."""
    c = np.asarray(counts, dtype=np.int64).reshape(-1, 3)
    res = {}
    for t, (tp, fp, fn) in zip(np.ravel(thresholds), c):
        den = int(tp + fp + fn)
        res[float(t)] = 1.0 if den == 0 else int(tp) / den
    return res


def ray_iou(pred, gt, origins=None, dirs=None, thresholds=DEFAULT_THRESHOLDS) -> dict:
    """RayIoU@t for SemanticGrids; rays default to
    ``default_rays(pred.spec)``."""
    _check_pair(pred, gt)
    if origins is None and dirs is None:
        origins, dirs = default_rays(pred.spec)
    C = len(pred.classes)
    p = _labels_u8(np.asarray(pred.labels).transpose(2, 1, 0), C, pred.classes.free_index)
    g = _labels_u8(np.asarray(gt.labels).transpose(2, 1, 0), C, gt.classes.free_index)
    cnt = ray_counts(p, g, pred.spec, C, origins, dirs, thresholds)
    return rayiou_from_counts(cnt.cpu().numpy(), thresholds)
