"""Cost of the live evaluator counters (sqv_stats_attach) and of the stage
profiler on the device-resident step (GPU box): run_many over K config-2
batches with each instrument on/off, interleaved, best of 3."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17361_b200 as P  # noqa: E402
from paper_2511_17361_b200 import _lib  # noqa: E402
from paper_2511_17361_b200.scenegen import gen_frames  # noqa: E402

vox = P.Voxelizer(P.VoxelGridSpec(), P.VoxelizeConfig(), 18)
dev = [vox.to_device(gen_frames(20251117 + 100 * k, 100, 2000, 18)) for k in range(4)]
outs = [vox.alloc(100), vox.alloc(100)]
st = torch.zeros(2, dtype=torch.int64, device="cuda")
K = 10


def run(stats, prof):
    _lib.stats_attach(st if stats else None)
    _lib.profile_enable(prof)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    vox.run_many([dev[k % 4] for k in range(K)], outs)
    e1.record()
    torch.cuda.synchronize()
    _lib.profile_read(reset=True)
    _lib.profile_enable(False)
    _lib.stats_attach(None)
    return e0.elapsed_time(e1) / K


run(False, False)
best = {}
for rep in range(4):
    for key in ((False, False), (True, False), (False, True), (True, True)):
        best[key] = min(best.get(key, 1e9), run(*key))
for (s, p), v in best.items():
    print(f"stats={s!s:5} profiler={p!s:5} ms/step {v:.3f}")
