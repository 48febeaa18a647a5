import sys, time, torch, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2511_17361_b200 as P
from paper_2511_17361_b200.scenegen import gen_frames
spec, cfg = P.VoxelGridSpec(), P.VoxelizeConfig()
vox = P.Voxelizer(spec, cfg, 18)
host = [gen_frames(1 + 100 * k, 100, 2000, 18) for k in range(4)]
pinned = [P.PrimitiveBatch(**{k: torch.from_numpy(np.ascontiguousarray(getattr(b, k))).pin_memory() for k in P.PrimitiveBatch.FIELDS}) for b in host]
labels = [torch.empty((100, 16, 200, 200), dtype=torch.uint8).pin_memory() for _ in range(40)]
vox.stream(pinned[:2], labels_out=labels[:2])
for K in (1, 2, 4, 8, 16, 32):
    seq = [pinned[k % 4] for k in range(K)]
    torch.cuda.synchronize()
    best = 1e9
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); vox.stream(seq, labels_out=labels[:K]); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(K, "ms %.2f" % best, "per step %.3f" % (best / K))
