"""End-to-end fixed cost of Voxelizer.stream (GPU box): t(K) for K pinned
100-frame config-2 batches, labels back to the host, with and without the
edge ranges (first/last batch split in frame ranges).  Best of 3 per point,
the two settings interleaved.  usage: python scripts/e2e_fixed_cost.py [edge piece counts, default 1,4]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17361_b200 as P  # noqa: E402
from paper_2511_17361_b200.scenegen import gen_frames  # noqa: E402

spec, cfg = P.VoxelGridSpec(), P.VoxelizeConfig()
vox = P.Voxelizer(spec, cfg, 18)
host = [gen_frames(1 + 100 * k, 100, 2000, 18) for k in range(4)]
pinned = [P.PrimitiveBatch(**{k: torch.from_numpy(np.ascontiguousarray(getattr(b, k))).pin_memory()
                              for k in P.PrimitiveBatch.FIELDS}) for b in host]
labels = [torch.empty((100, 16, 200, 200), dtype=torch.uint8).pin_memory() for _ in range(20)]
dev = [vox.to_device(b) for b in pinned]
outs = [vox.alloc(100), vox.alloc(100)]
EDGES = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 4]
for e in EDGES:
    vox.stream(pinned[:2], labels_out=labels[:2], edge_pieces=e)
vox.run_many(dev[:2], outs)
torch.cuda.synchronize()


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


for K in (1, 2, 4, 10, 20):
    seq = [pinned[k % 4] for k in range(K)]
    d = timed(lambda: vox.run_many([dev[k % 4] for k in range(K)], outs))
    row = {"K": K, "device_resident_ms": round(d, 3)}
    for e in EDGES:
        row[f"edge{e}_ms"] = round(timed(lambda: vox.stream(seq, labels_out=labels[:K],
                                                             edge_pieces=e)), 3)
    print(row, flush=True)
