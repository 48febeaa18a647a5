"""Accumulation-depth diagnostic: v_o error vs the oracle as a function of
entries per tile (TC vs FFMA evaluator).  Writes gpurun_out/diag_depth.json."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17361_b200 as P
from paper_2511_17361_b200.scenegen import gen_frames
from oracle import oracle as O

out = []
for N, dims, res in [(2000, (200, 200, 16), 0.4), (600, (48, 48, 16), 0.4),
                     (1200, (48, 48, 16), 0.4), (2400, (48, 48, 16), 0.4)]:
    origin = (-dims[0] * res / 2, -dims[1] * res / 2, -1.0)
    spec = P.VoxelGridSpec(origin, dims, res)
    b = gen_frames(3, 1, N, 18, origin=origin, dims=dims, resolution=res)
    p = O.Prims.of(b)
    g = O.Grid(origin, dims, res)
    row = {"N": N, "dims": dims}
    for ev in ("tc", "ffma"):
        os.environ["SQV_EVAL"] = ev
        vox = P.Voxelizer(spec, P.VoxelizeConfig(), 18)
        r = vox(b, dense=True)
        vo = r.v_o.reshape(-1).cpu().numpy().astype(np.float64)
        if ev == "tc":
            ref = O.voxelize(p, g, O.Cfg(free_label=r.free_code))
            rv = ref["v_o"].reshape(-1)
            row["entries_per_tile"] = r.n_entries / vox.tiles_per_frame
        rel = np.abs(vo - rv) / np.maximum(rv, 1e-5)
        row[ev] = {"max": float(rel.max()), "p99": float(np.quantile(rel, 0.99)),
                   "mean_signed": float(np.mean((vo - rv) / np.maximum(rv, 1e-5)))}
    os.environ.pop("SQV_EVAL", None)
    out.append(row)
    print(row, flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/diag_depth.json", "w"), indent=1)
