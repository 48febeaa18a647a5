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
