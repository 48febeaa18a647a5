"""A/B of Voxelizer.stream variants (GPU box): t(K) for K pinned 100-frame
batches of a bench config, labels back to the host, best of 3, interleaved."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2511_17361_b200 as P  # noqa: E402
from paper_2511_17361_b200.scenegen import gen_frames  # noqa: E402
import diag_stream_old  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
vox = P.Voxelizer(P.VoxelGridSpec(), P.VoxelizeConfig(), 18)
host = [gen_frames(1 + 100 * k, 100, N, 18) for k in range(4)]
pinned = [P.PrimitiveBatch(**{k: torch.from_numpy(np.ascontiguousarray(getattr(b, k))).pin_memory()
                              for k in P.PrimitiveBatch.FIELDS}) for b in host]
labels = [torch.empty((100, 16, 200, 200), dtype=torch.uint8).pin_memory() for _ in range(20)]
dev = [vox.to_device(b) for b in pinned]
outs = [vox.alloc(100), vox.alloc(100)]
V = {"new_e4": lambda seq, K: vox.stream(seq, labels_out=labels[:K], edge_pieces=4),
     "new_e1": lambda seq, K: vox.stream(seq, labels_out=labels[:K], edge_pieces=1),
     "old": lambda seq, K: diag_stream_old.stream(vox, seq, labels_out=labels[:K])}
for f in V.values():
    f(pinned[:3], 3)
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


for K in (4, 20):
    seq = [pinned[k % 4] for k in range(K)]
    row = {"N": N, "K": K, "device": round(timed(lambda: vox.run_many([dev[k % 4] for k in range(K)], outs)), 3)}
    for name, f in V.items():
        row[name] = round(timed(lambda: f(seq, K)), 3)
    print(row, flush=True)
