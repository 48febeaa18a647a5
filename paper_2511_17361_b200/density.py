"""Point-wise density on the device: ``inside_outside`` / ``density`` of
core.py:254-282 for many (primitive, world point) pairs (include/sqv.h
``sqv_density``).  Same FP32 SFU field as the voxel evaluator, FP64 setup and
transform.  F is reported capped at F_CAP like the reference; density is 0
where FP32 exp(-F) underflows (F >= 87.3365).
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .core import PrimitiveBatch


def density_pairs(batch: PrimitiveBatch, points, pair_prim):
    """(F, density) float32 numpy arrays for point k against primitive
    pair_prim[k] of a one-frame batch."""
    import torch
    dev = _lib.require_cuda()
    L = _lib.lib()
    if batch.n_frames != 1:
        raise ValueError("density_pairs takes a one-frame batch")
    t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt).to(dev)
    mu, scale, rot = (t(getattr(batch, k), torch.float64) for k in ("mu", "scale", "rot"))
    opacity, eps, logits = (t(getattr(batch, k), torch.float64)
                            for k in ("opacity", "eps", "logits"))
    pts = t(np.asarray(points, np.float64).reshape(-1, 3), torch.float64)
    pp = t(np.asarray(pair_prim, np.int32).ravel(), torch.int32)
    n = pts.shape[0]
    if pp.numel() != n:
        raise ValueError("points and pair_prim lengths differ")
    P = _lib.Prims()
    P.mu, P.scale, P.rot = mu.data_ptr(), scale.data_ptr(), rot.data_ptr()
    P.opacity, P.eps, P.logits = opacity.data_ptr(), eps.data_ptr(), logits.data_ptr()
    P.n_valid = None
    P.n_frames, P.n_prims, P.n_classes = 1, batch.n_prims, batch.n_classes
    F = torch.empty(n, dtype=torch.float32, device=dev)
    d = torch.empty(n, dtype=torch.float32, device=dev)
    import ctypes
    _lib.check(L.sqv_density(ctypes.byref(P), pts.data_ptr(), pp.data_ptr(), n, F.data_ptr(),
                             d.data_ptr(), _lib.stream_ptr(dev)), "sqv_density")
    return F.cpu().numpy(), d.cpu().numpy()
