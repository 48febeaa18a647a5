"""Stage timelines (SQV_PROF_TRACE=1) of run_many on device batches and of
Voxelizer.stream on pinned host batches (GPU box, diagnostics): per call,
the prep, scan, readback, masks and evaluator events on one clock (stderr).
usage: SQV_PROF_TRACE=1 python scripts/diag_e2e_trace.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17361_b200 as P
from paper_2511_17361_b200 import _lib
from paper_2511_17361_b200.scenegen import gen_frames
vox = P.Voxelizer(P.VoxelGridSpec(), P.VoxelizeConfig(), 18)
host = [gen_frames(1 + 100 * k, 100, 2000, 18) for k in range(4)]
pinned = [P.PrimitiveBatch(**{k: torch.from_numpy(np.ascontiguousarray(getattr(b, k))).pin_memory() for k in P.PrimitiveBatch.FIELDS}) for b in host]
labels = [torch.empty((100, 16, 200, 200), dtype=torch.uint8).pin_memory() for _ in range(8)]
dev = [vox.to_device(b) for b in pinned]
outs = [vox.alloc(100), vox.alloc(100)]
vox.stream(pinned[:2], labels_out=labels[:2], edge_pieces=1)
vox.run_many(dev[:2], outs)
torch.cuda.synchronize()
K = 6
for name, fn in (("run_many", lambda: vox.run_many([dev[k % 4] for k in range(K)], outs)),
                 ("stream", lambda: vox.stream([pinned[k % 4] for k in range(K)], labels_out=labels[:K], edge_pieces=1)),
                 ("stream_nolab", lambda: vox.stream([dev[k % 4] for k in range(K)], labels_out=labels[:K], edge_pieces=1))):
    torch.cuda.synchronize()
    print("==", name, file=sys.stderr, flush=True)
    _lib.profile_enable(True); _lib.profile_read(reset=True)
    fn(); torch.cuda.synchronize()
    _lib.profile_read(reset=True); _lib.profile_enable(False)
