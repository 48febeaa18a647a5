"""Multi-GPU: frame sharding and the confusion-count all-reduce.

Frames are independent, so ranks own contiguous frame blocks
and never exchange voxel data.  The only collective on the path is one
SUM all-reduce of the int64 (C+1)^2 confusion counts — NCCL over NVLink on
B200 (process group backend "nccl"), gloo in the CPU tests.  Integer sums are
exact, so the global counts (and hence IoU/mIoU) are bit-identical for any
GPU count.
"""
from __future__ import annotations

import os


def shard_frames(n_frames: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [start, stop) block of frames for `rank` (first n % world
    ranks take one extra frame)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("invalid rank/world")
    base, extra = divmod(int(n_frames), world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def env_rank_world() -> tuple[int, int, int]:
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def allreduce_confusion(cm, group=None):
    """In-place SUM all-reduce of an int64 count tensor (no-op single process)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(cm, op=dist.ReduceOp.SUM, group=group)
    return cm


def evaluate_stream(voxelizer, batches, gt_labels, n_classes: int, group=None):
    """Voxelize this rank's frame batches, accumulate confusion counts against
    device-resident ground-truth labels (list of uint8 tensors, one per batch),
    all-reduce once at the end.  Returns the global (C+1)^2 counts (device)."""
    import torch
    from .metrics import confusion_matrix
    K = n_classes + 1
    cm = torch.zeros((K, K), dtype=torch.int64, device=voxelizer.device)
    for batch, gt in zip(batches, gt_labels):
        r = voxelizer(batch, dense=False)
        confusion_matrix(r.labels, gt, n_classes, out=cm)
    return allreduce_confusion(cm, group)


def gt_jitter_device(gt_seed: int, first_frame: int, n_frames: int, n_prims: int,
                     n_classes: int, device=None):
    """Per-frame N(0, 1) jitter draws for the ground-truth copy of frames
    first_frame .. first_frame+n_frames-1: (d_mu [F, N, 3], d_logits [F, N, C]).

    They come from the same counter-based Philox stream as the scenes
    (``sqv_gen_frames`` keyed by gt_seed: its C + 3 standard normals per
    primitive, the first 3 for mu, the rest for the logits), so the draws of
    a frame depend only on (gt_seed, frame, primitive): never on the batch
    size or the rank's shard.  The confusion counts are therefore identical
    for any frames_per_batch and any GPU count."""
    from .scenegen import gen_frames_device
    z = gen_frames_device(gt_seed, n_frames, n_prims, n_classes + 3,
                          first_frame=first_frame, device=device).logits
    return z[..., :3], z[..., 3:]


def evaluate_generated(voxelizer, seed: int, n_frames: int, n_prims: int,
                       frames_per_batch: int = 100, gt_seed: int | None = None,
                       sigma_mu: float = 0.2, sigma_logit: float = 0.5, smin: float = 0.2,
                       smax: float = 4.0, emin: float = 0.2, group=None,
                       frame_range: tuple[int, int] | None = None):
    """The config-5 stream with no host in the loop: this rank's frame shard
    is generated in HBM (``scenegen.gen_frames_device``: frame f depends only
    on (seed, f), so shards need no coordination), the ground truth is a
    jittered copy (mu + N(0, sigma_mu), logits + N(0, sigma_logit), drawn
    per frame by ``gt_jitter_device``), both are voxelized and their
    confusion counts accumulated, then all-reduced once.  Returns the global
    counts, bit-identical for any frames_per_batch and world size.
    ``frame_range`` overrides this rank's shard (default ``shard_frames``)."""
    import torch
    import torch.distributed as dist
    from .core import PrimitiveBatch
    from .metrics import confusion_matrix
    from .scenegen import gen_frames_device
    if dist.is_available() and dist.is_initialized():
        rank, world = dist.get_rank(group), dist.get_world_size(group)
    else:
        rank, world = 0, 1
    C = voxelizer.C
    spec = voxelizer.spec
    dev = voxelizer.device
    gt_seed = seed + 1 if gt_seed is None else gt_seed
    K = C + 1
    cm = torch.zeros((K, K), dtype=torch.int64, device=dev)
    start, stop = frame_range if frame_range is not None else shard_frames(n_frames, rank, world)
    for f0 in range(start, stop, frames_per_batch):
        F = min(frames_per_batch, stop - f0)
        b = gen_frames_device(seed, F, n_prims, C, origin=spec.origin, dims=spec.dims,
                              resolution=spec.resolution, smin=smin, smax=smax, emin=emin,
                              first_frame=f0, device=dev)
        d_mu, d_lg = gt_jitter_device(gt_seed, f0, F, n_prims, C, device=dev)
        gt = PrimitiveBatch(b.mu + sigma_mu * d_mu, b.scale, b.rot, b.opacity, b.eps,
                            b.logits + sigma_logit * d_lg)
        pred_l = voxelizer(b, dense=False).labels
        gt_l = voxelizer(gt, dense=False).labels
        confusion_matrix(pred_l, gt_l, C, out=cm)
    return allreduce_confusion(cm, group)
