"""Where the strict-mode v_o error tail comes from (GPU box, diagnostics):
config-1 frames (bench seed), every voxel with |dv_o| / max(v_o, 1e-5)
above a threshold, and for the worst ones the primitives that reach the
voxel: sigma, eps1 (c = 2/eps1), F and share of v_o (FP64 oracle, the
checker).  Run it under several libraries (SQV_LIB=variants/...) to see
which arithmetic closes the tail.
usage: python scripts/diag_precision_tail.py FRAMES [THRESH] [frame list]"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_17361_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2511_17361_b200.scenegen import gen_frames  # noqa: E402

SEED, N = 20251117, 256
F = int(sys.argv[1]) if len(sys.argv) > 1 else 64
TH = float(sys.argv[2]) if len(sys.argv) > 2 else 8e-6
only = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else None
spec = P.VoxelGridSpec()
grid = O.Grid(spec.origin, spec.dims, spec.resolution)
vox = P.Voxelizer(spec, P.VoxelizeConfig(precision="strict"), 18, free_index=255)
frames = only if only is not None else list(range(F))
hits = []
for f0 in range(0, len(frames), 64):
    fl = frames[f0:f0 + 64]
    bs = [gen_frames(SEED, 1, N, 18, first_frame=f) for f in fl]
    for f, b in zip(fl, bs):
        ref = O.voxelize(O.Prims.of(b), grid, O.Cfg(free_label=255), want_vc=False)["v_o"][0]
        got = vox(b, dense=True).v_o.reshape(-1).cpu().numpy().astype(np.float64)
        rel = np.abs(got - ref) / np.maximum(ref, 1e-5)
        for v in np.flatnonzero(rel > TH):
            hits.append((float(rel[v]), f, int(v), float(ref[v]), float(got[v])))
hits.sort(reverse=True)
print("voxels above", TH, ":", len(hits))
nx, ny, nz = spec.dims
for rel, f, v, ref, got in hits[:8]:
    b = gen_frames(SEED, 1, N, 18, first_frame=f)
    p = O.Prims.of(b)
    win = O.prep(p, grid, O.Cfg(free_label=255))[0]
    x, y, z = v % nx, (v // nx) % ny, v // (nx * ny)
    inside = np.flatnonzero((win[:, 0] <= x) & (x <= win[:, 3]) & (win[:, 1] <= y) &
                            (y <= win[:, 4]) & (win[:, 2] <= z) & (z <= win[:, 5]))
    pt = np.asarray(spec.origin) + (np.array([x, y, z]) + 0.5) * spec.resolution
    Fv, dv = O.density(p, np.repeat(pt[None], len(inside), 0), inside.astype(np.int32))
    sig = p.opacity[0, inside]
    contrib = sig * dv
    eps = np.clip(p.eps[0, inside], 0.2, 2.0)
    order = np.argsort(-contrib)
    print(json.dumps({"rel": rel, "frame": f, "voxel": [x, y, z], "v_o": ref, "gpu": got}))
    for k in order[:4]:
        print(f"   prim {inside[k]:4d} sigma {sig[k]:.3f} eps1 {eps[k, 0]:.3f} eps2 {eps[k, 1]:.3f}"
              f" c {2 / eps[k, 0]:.2f} a {2 / eps[k, 1]:.2f} F {Fv[k]:8.4f} share {contrib[k] / ref:.4f}")
