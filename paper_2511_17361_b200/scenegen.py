"""Seeded synthetic scenes (SPEC.md:594-597 ``gen_scene``), vectorised.

The reference specifies gen_scene only as text: "deterministic pseudo-random
primitives inside the grid bounds with scales in [0.2, 4.0] m, eps in clamp
range, logits from a seeded draw".  This module pins one generator (the one
BASELINE.md / SURVEY.md §8d define the benchmark on):

  rng = numpy.random.default_rng(seed + frame)            (PCG64)
  mu      ~ U(grid bounds)^3           rng.uniform(lo, hi, (N, 3))
  scale   ~ U[smin, smax]^3            rng.uniform(smin, smax, (N, 3))
  rot     = normal(0,1)^4, normalised  (random_unit_quat, core.py:102-106)
  opacity ~ U[0, 1]                    rng.uniform(0, 1, N)
  eps     ~ U[emin, 2.0]^2             rng.uniform(emin, 2.0, (N, 2))
  logits  ~ N(0, 1)^C                  rng.normal(size=(N, C))

drawn in exactly that order.  ``emin`` = 0.1 gives the stress set of config 3
(clamped to 0.2 on the device, core.py:162-165); ``smax`` = 1.0 gives the
sparse variant that leaves free space and exercises tau.
"""
from __future__ import annotations

import numpy as np

from .core import PrimitiveBatch


def _frame(rng, n, C, lo, hi, smin, smax, emin):
    mu = rng.uniform(lo, hi, size=(n, 3))
    scale = rng.uniform(smin, smax, size=(n, 3))
    q = rng.normal(size=(n, 4))
    nq = np.linalg.norm(q, axis=1)
    while np.any(nq < 1e-6):  # random_unit_quat's rejection loop, core.py:103-105
        bad = nq < 1e-6
        q[bad] = rng.normal(size=(int(bad.sum()), 4))
        nq = np.linalg.norm(q, axis=1)
    rot = q / nq[:, None]
    opacity = rng.uniform(0.0, 1.0, size=n)
    eps = rng.uniform(emin, 2.0, size=(n, 2))
    logits = rng.normal(size=(n, C))
    return mu, scale, rot, opacity, eps, logits


def gen_frames(seed: int, n_frames: int, n_prims: int, n_classes: int = 18,
               origin=(-40.0, -40.0, -1.0), dims=(200, 200, 16), resolution: float = 0.4,
               smin: float = 0.2, smax: float = 4.0, emin: float = 0.2,
               first_frame: int = 0) -> PrimitiveBatch:
    """Frames first_frame .. first_frame+n_frames-1 of the seeded stream."""
    lo = np.asarray(origin, np.float64)
    hi = lo + np.asarray(dims, np.float64) * float(resolution)
    F, N, C = n_frames, n_prims, n_classes
    out = [np.empty((F, N, 3)), np.empty((F, N, 3)), np.empty((F, N, 4)), np.empty((F, N)),
           np.empty((F, N, 2)), np.empty((F, N, C))]
    for f in range(F):
        rng = np.random.default_rng(seed + first_frame + f)
        for dst, src in zip(out, _frame(rng, N, C, lo, hi, smin, smax, emin)):
            dst[f] = src
    return PrimitiveBatch(*out)


def gen_scene(seed: int, n: int, n_classes: int = 18, **grid) -> PrimitiveBatch:
    """One frame (SPEC.md:594 gen_scene(seed, n, grid spec))."""
    return gen_frames(seed, 1, n, n_classes, **grid)


def jitter(batch: PrimitiveBatch, seed: int, sigma_mu: float = 0.2,
           sigma_logit: float = 0.5) -> PrimitiveBatch:
    """Perturbed copy (ground-truth stand-in for the mIoU stream, SURVEY.md §8d
    config 5): mu += N(0, sigma_mu), logits += N(0, sigma_logit)."""
    rng = np.random.default_rng(seed)
    mu = np.asarray(batch.mu) + rng.normal(scale=sigma_mu, size=np.shape(batch.mu))
    logits = np.asarray(batch.logits) + rng.normal(scale=sigma_logit,
                                                   size=np.shape(batch.logits))
    return PrimitiveBatch(mu, np.asarray(batch.scale), np.asarray(batch.rot),
                          np.asarray(batch.opacity), np.asarray(batch.eps), logits,
                          n_valid=batch.n_valid)


def gen_frames_device(seed: int, n_frames: int, n_prims: int, n_classes: int = 18,
                      origin=(-40.0, -40.0, -1.0), dims=(200, 200, 16), resolution: float = 0.4,
                      smin: float = 0.2, smax: float = 4.0, emin: float = 0.2,
                      first_frame: int = 0, device=None, stream=None) -> PrimitiveBatch:
    """The same distributions generated in HBM by the ``sqv_gen_frames``
    kernel (Philox4x32-10 counter stream; include/sqv.h): a PrimitiveBatch of
    device tensors, ready for ``Voxelizer``.  A different (counter-based)
    stream than ``gen_frames``: frame f of (seed, first_frame) depends only on
    seed and first_frame + f, so ranks generate their own shards."""
    import ctypes

    import torch

    from . import _lib
    from .voxelize import VoxelGridSpec
    dev = _lib.require_cuda() if device is None else torch.device(device)
    L = _lib.lib()
    if not (0 <= seed < 2 ** 64):
        raise ValueError("seed must be a 64-bit unsigned integer")
    F, N, C = int(n_frames), int(n_prims), int(n_classes)
    mk = lambda *s: torch.empty((F, N) + s, dtype=torch.float64, device=dev)
    mu, scale, rot, opacity, eps, logits = mk(3), mk(3), mk(4), mk(), mk(2), mk(C)
    g = VoxelGridSpec(origin=tuple(origin), dims=tuple(dims), resolution=resolution)._c()
    s = stream if stream is not None else _lib.stream_ptr(dev)
    with torch.cuda.device(dev):
        _lib.check(L.sqv_gen_frames(int(seed), int(first_frame), F, N, C, ctypes.byref(g),
                                    float(smin), float(smax), float(emin), mu.data_ptr(),
                                    scale.data_ptr(), rot.data_ptr(), opacity.data_ptr(),
                                    eps.data_ptr(), logits.data_ptr(), s), "sqv_gen_frames")
    return PrimitiveBatch(mu, scale, rot, opacity, eps, logits)
