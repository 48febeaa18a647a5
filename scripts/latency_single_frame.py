"""Single-frame latency (the paper's inference use: one frame of N
superquadrics at a time): device-resident inputs ->
labels on the device, and the drop-in voxelize() from host inputs to host
grids.  Median of 50 calls after warm-up."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_17361_b200 as P  # noqa: E402
from paper_2511_17361_b200.scenegen import gen_frames  # noqa: E402

spec = P.VoxelGridSpec()
for n in (256, 1600, 2000):
    vox = P.Voxelizer(spec, P.VoxelizeConfig(), 18)
    b = vox.to_device(gen_frames(5, 1, n, 18))
    out = vox.alloc(1, dense=False)
    for _ in range(5):
        vox(b, dense=False, out=out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(50):
        t0 = time.perf_counter()
        vox(b, dense=False, out=out)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    dev_ms = 1e3 * float(np.median(ts))
    hb = gen_frames(6, 1, n, 18)
    outd = vox.alloc(1, dense=True)
    for _ in range(3):
        r = vox(hb, dense=True, out=outd)
        r.labels.cpu()
    ts = []
    for _ in range(20):
        t0 = time.perf_counter()
        r = vox(hb, dense=True, out=outd)
        lab = r.labels.cpu()
        ts.append(time.perf_counter() - t0)
    host_ms = 1e3 * float(np.median(ts))
    print(f"N={n}: device inputs -> device labels {dev_ms:.3f} ms; host inputs -> host labels "
          f"(dense grids on device) {host_ms:.3f} ms")
