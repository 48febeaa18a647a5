"""``torch.ops.sqocc.*`` — the PyTorch-operator face of libsqv (SURVEY.md §3(4),
§8(b): "a PyTorch extension registering torch.ops.sqocc.{prep_bin, voxelize,
confusion}").

Importing this module registers three custom operators (``torch.library``)
over the same C ABI the rest of the package calls (include/sqv.h); they run
on the current CUDA stream and have fake (meta) implementations, so they
trace under FakeTensor / ``torch.compile`` like any other op:

* ``sqocc::voxelize(mu, scale, rot, opacity, eps, logits, origin, dims,
  resolution, tau, neighborhood_radius, semantic_mode, precision, truncate,
  free_index) -> (labels, v_o, v_c)`` — SPEC.md:345-373 on F frames of N
  primitives (FP64 SoA: mu/scale [F,N,3], rot [F,N,4], opacity [F,N],
  eps [F,N,2], logits [F,N,C]).  labels uint8 [F,nz,ny,nx] (free voxels =
  ``free_index`` if it fits a byte, else 255), v_o float32 [F,nz,ny,nx],
  v_c float32 [F,nz,ny,nx,C] — x-fastest memory.
  ``truncate=False`` is ``voxelize_bruteforce``.
* ``sqocc::prep_bin(mu, ..., truncate) -> (windows, tile_off, prim_ids,
  n_pairs)`` — the bins: per-primitive clipped windows
  int32 [F,N,6], tile offsets int32 [F*T+1] and ascending primitive ids
  int32 [E] per 8x8x16 tile, the algorithmic pair count int64 [].  E is data
  dependent (an unbacked size under FakeTensor).
* ``sqocc::confusion(pred, gt, n_classes) -> cm`` — SPEC.md:494-512 counts,
  int64 [(C+1), (C+1)], row = gt, column = pred, labels >= C free.

There is no CPU kernel: a CPU tensor raises (no fallback, like every entry
point of the package).
"""
from __future__ import annotations

import torch
from torch import Tensor

from .voxelize import (PRECISIONS, SEMANTIC_MODES, VoxelGridSpec, VoxelizeConfig, Voxelizer,
                       free_code_for)

_VOXELIZERS: dict = {}  # (grid, config, C, free index, device) -> Voxelizer (its workspaces)
_MAX_CACHED = 16


def _voxelizer(origin, dims, resolution, tau, radius, mode, precision, truncate, C, free_index,
               device) -> Voxelizer:
    key = (tuple(origin), tuple(dims), float(resolution), float(tau), int(radius), mode, precision,
           bool(truncate), int(C), int(free_index), str(device))
    v = _VOXELIZERS.get(key)
    if v is None:
        if mode not in SEMANTIC_MODES:
            raise ValueError(f"semantic_mode must be one of {SEMANTIC_MODES}")
        if precision not in PRECISIONS:
            raise ValueError(f"precision must be one of {PRECISIONS}")
        spec = VoxelGridSpec(tuple(origin), tuple(dims), resolution)
        cfg = VoxelizeConfig(tau=tau, neighborhood_radius=radius, semantic_mode=mode,
                             precision=precision)
        v = Voxelizer(spec, cfg, C, None if free_index < 0 else free_index, truncate=truncate,
                      device=device)
        if len(_VOXELIZERS) >= _MAX_CACHED:  # bounded: drop the oldest configuration
            _VOXELIZERS.pop(next(iter(_VOXELIZERS)))
        _VOXELIZERS[key] = v
    return v


def _batch(mu, scale, rot, opacity, eps, logits):
    from .core import PrimitiveBatch
    for t in (mu, scale, rot, opacity, eps, logits):
        if not t.is_cuda:
            raise RuntimeError("torch.ops.sqocc.* run on CUDA tensors only (no CPU fallback)")
    return PrimitiveBatch(mu, scale, rot, opacity, eps, logits)


def _check_shapes(mu, scale, rot, opacity, eps, logits):
    if mu.dim() != 3 or mu.shape[-1] != 3:
        raise ValueError("mu must be [F, N, 3]")
    F, N = mu.shape[0], mu.shape[1]
    for name, t, tail in (("scale", scale, (3,)), ("rot", rot, (4,)), ("opacity", opacity, ()),
                          ("eps", eps, (2,))):
        if tuple(t.shape) != (F, N) + tail:
            raise ValueError(f"{name} must be [F, N{', ' + str(tail[0]) if tail else ''}]")
    if logits.dim() != 3 or tuple(logits.shape[:2]) != (F, N):
        raise ValueError("logits must be [F, N, C]")
    return F, N, logits.shape[2]


@torch.library.custom_op("sqocc::voxelize", mutates_args=())
def voxelize_op(mu: Tensor, scale: Tensor, rot: Tensor, opacity: Tensor, eps: Tensor,
                logits: Tensor, origin: list[float], dims: list[int], resolution: float,
                tau: float = 0.01, neighborhood_radius: int = 5, semantic_mode: str = "logit-sum",
                precision: str = "strict", truncate: bool = True,
                free_index: int = -1) -> tuple[Tensor, Tensor, Tensor]:
    F, N, C = _check_shapes(mu, scale, rot, opacity, eps, logits)
    vox = _voxelizer(origin, dims, resolution, tau, neighborhood_radius, semantic_mode, precision,
                     truncate, C, free_index, mu.device)
    r = vox(_batch(mu, scale, rot, opacity, eps, logits), dense=True)
    return r.labels, r.v_o, r.v_c


@voxelize_op.register_fake
def _(mu, scale, rot, opacity, eps, logits, origin, dims, resolution, tau=0.01,
      neighborhood_radius=5, semantic_mode="logit-sum", precision="strict", truncate=True,
      free_index=-1):
    F, N, C = _check_shapes(mu, scale, rot, opacity, eps, logits)
    nx, ny, nz = (int(d) for d in dims)
    return (mu.new_empty((F, nz, ny, nx), dtype=torch.uint8),
            mu.new_empty((F, nz, ny, nx), dtype=torch.float32),
            mu.new_empty((F, nz, ny, nx, C), dtype=torch.float32))


@torch.library.custom_op("sqocc::prep_bin", mutates_args=())
def prep_bin_op(mu: Tensor, scale: Tensor, rot: Tensor, opacity: Tensor, eps: Tensor,
                logits: Tensor, origin: list[float], dims: list[int], resolution: float,
                neighborhood_radius: int = 5, truncate: bool = True
                ) -> tuple[Tensor, Tensor, Tensor, Tensor]:
    F, N, C = _check_shapes(mu, scale, rot, opacity, eps, logits)
    vox = _voxelizer(origin, dims, resolution, 0.01, neighborhood_radius, "logit-sum", "strict",
                     truncate, C, -1, mu.device)
    # the bins come out of the same sqv_voxelize call (labels only, dense
    # grids never leave the chip)
    r = vox(_batch(mu, scale, rot, opacity, eps, logits), dense=False, bins=True)
    n_pairs = torch.tensor(r.n_pairs, dtype=torch.int64, device=mu.device)
    return (r.bins["windows"], r.bins["tile_off"], r.bins["prim_ids"].clone(), n_pairs)


@prep_bin_op.register_fake
def _(mu, scale, rot, opacity, eps, logits, origin, dims, resolution, neighborhood_radius=5,
      truncate=True):
    F, N, C = _check_shapes(mu, scale, rot, opacity, eps, logits)
    T = 1
    for d, t in zip(dims, (8, 8, 16)):  # SQV_TILE_X/Y/Z (include/sqv.h)
        T *= (int(d) + t - 1) // t
    E = torch.library.get_ctx().new_dynamic_size()
    return (mu.new_empty((F, N, 6), dtype=torch.int32),
            mu.new_empty((F * T + 1,), dtype=torch.int32),
            mu.new_empty((E,), dtype=torch.int32),
            mu.new_empty((), dtype=torch.int64))


@torch.library.custom_op("sqocc::confusion", mutates_args=())
def confusion_op(pred: Tensor, gt: Tensor, n_classes: int) -> Tensor:
    from .metrics import confusion_matrix
    if not (pred.is_cuda and gt.is_cuda):
        raise RuntimeError("torch.ops.sqocc.confusion runs on CUDA tensors only")
    if pred.dtype != torch.uint8 or gt.dtype != torch.uint8:
        raise ValueError("labels must be uint8")
    return confusion_matrix(pred, gt, n_classes)


@confusion_op.register_fake
def _(pred, gt, n_classes):
    if pred.numel() != gt.numel():
        raise ValueError("dimension mismatch")
    K = int(n_classes) + 1
    return pred.new_empty((K, K), dtype=torch.int64)


__all__ = ["voxelize_op", "prep_bin_op", "confusion_op", "free_code_for"]
