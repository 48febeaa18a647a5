"""Config 5 (BASELINE.json): the 6,019-frame val-sized synthetic stream with
the mIoU confusion counts, run through distributed.evaluate_generated — scenes
generated in HBM (sqv_gen_frames), a per-frame jittered copy as ground truth,
both voxelized, int64 confusion counts accumulated on the device and
all-reduced (a no-op at one GPU; NCCL under torchrun).  Prints one JSON line:
frames/s of the stream (two voxelizations per frame), IoU and mIoU.

usage: python scripts/config5_stream.py [n_frames] [frames_per_batch]
   or: torchrun --nproc-per-node N scripts/config5_stream.py ...
"""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_17361_b200 as P  # noqa: E402
from paper_2511_17361_b200 import distributed as D  # noqa: E402
from paper_2511_17361_b200.metrics import iou_from_confusion, miou_from_confusion  # noqa: E402


def main():
    n_frames = int(sys.argv[1]) if len(sys.argv) > 1 else 6019
    fpb = int(sys.argv[2]) if len(sys.argv) > 2 else 100
    rank, world, local = D.env_rank_world()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    vox = P.Voxelizer(P.VoxelGridSpec(), P.VoxelizeConfig(), 18)
    D.evaluate_generated(vox, 11, 2 * fpb, 2000, frames_per_batch=fpb)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cm = D.evaluate_generated(vox, 20251117, n_frames, 2000, frames_per_batch=fpb)
    cm_host = cm.cpu().numpy()
    dt = time.perf_counter() - t0
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([dt], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    if rank == 0:
        per, m, _ = miou_from_confusion(cm_host)
        print(json.dumps({"workload": "config5: 6,019-frame synthetic stream, 2k SQs/frame, "
                                      "200x200x16, pred + jittered gt voxelized per frame",
                          "n_gpus": world, "frames": n_frames, "frames_per_batch": fpb,
                          "wall_s": dt, "frames_per_s": n_frames / dt,
                          "voxelizations_per_s": 2 * n_frames / dt,
                          "confusion_total": int(cm_host.sum()),
                          "iou": iou_from_confusion(cm_host), "miou": m}))


if __name__ == "__main__":
    main()
