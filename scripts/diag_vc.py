"""v_c error vs the oracle under the parity scale max(|v_c|, v_o, 1e-3) (and
1e-3 tau floor variants) on config-1/2 frames, strict and fast."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17361_b200 as P
from paper_2511_17361_b200.scenegen import gen_frames
from oracle import oracle as O
res = {}
for N in (256, 2000):
    b = gen_frames(5, 1, N)
    spec = P.VoxelGridSpec()
    p = O.Prims.of(b)
    g = O.Grid(spec.origin, spec.dims, spec.resolution)
    for prec in ("strict", "fast"):
        r = P.Voxelizer(spec, P.VoxelizeConfig(precision=prec), 18)(b, dense=True)
        ref = O.voxelize(p, g, O.Cfg(free_label=r.free_code))
        vc = r.v_c.reshape(-1, 18).cpu().numpy().astype(np.float64)
        vr = ref["v_c"].reshape(-1, 18)
        vo = ref["v_o"].reshape(-1, 1)
        scale = np.maximum(np.maximum(np.abs(vr).max(1, keepdims=True), vo), 1e-3)
        rel = np.abs(vc - vr) / scale
        res[f"N{N}_{prec}"] = {"max": float(rel.max()), "p999": float(np.quantile(rel, 0.999))}
        print(N, prec, res[f"N{N}_{prec}"], flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/diag_vc.json", "w"), indent=1)
