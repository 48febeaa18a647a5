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

RayIoU is outside this round's scope.
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
