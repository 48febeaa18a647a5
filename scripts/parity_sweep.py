"""Parity at the benchmark's sizes over many frames (GPU box): the bench
configs' own generator (scenegen.gen_frames, the bench seed and grids)
voxelized by the product path in both precisions, every frame checked in
full against the FP64 oracle (oracle/, the checker): bins and pair counts
exact, the worst |dv_o| / max(v_o, floor), the worst v_c error against the
voxel's weight scale (with the term magnitudes sum_i w_i |c_ik| from an
oracle run on |logits|), label agreement and unexplained mismatches
(tests/parity.py rules).  Frames run in chunks (the oracle's FP64 v_c of a
config-4 frame is 0.7 GB).  Writes gpurun_out/parity_sweep.json.

usage: python scripts/parity_sweep.py [frames_c2] [frames_c3] [frames_c1] [frames_c4]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2511_17361_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2511_17361_b200.scenegen import gen_frames  # noqa: E402
from parity import VO_REL, VO_REL_TAIL, label_check, vo_check, weight_scale  # noqa: E402

SEED = 20251117  # bench.py default
OCC = dict(origin=(-40.0, -40.0, -1.0), dims=(200, 200, 16), resolution=0.4)
BIG = dict(origin=(-40.0, -40.0, -1.0), dims=(400, 400, 32), resolution=0.2)
arg = lambda i, d: int(sys.argv[i]) if len(sys.argv) > i else d
CONFIGS = {  # name: (frames, chunk, n_prims, grid, gen kwargs) — bench.py WORKLOADS
    "config2": (arg(1, 16), 16, 2000, OCC, {}),
    "config3": (arg(2, 4), 8, 4000, OCC, {"emin": 0.1}),
    "config1": (arg(3, 16), 32, 256, OCC, {}),
    "config4": (arg(4, 1), 1, 8000, BIG, {}),
}


def vc_worst(vc_g, vc_r, vo_r, tau, vc_abs):
    scale = weight_scale(vo_r, vc_r, tau, vc_abs).reshape(vc_r.shape[:-1])
    return float((np.abs(vc_g.astype(np.float64) - vc_r).max(axis=-1) / scale).max(initial=0.0))


def main():
    out = {"oracle_threads": O.threads(), "configs": {}}
    for name, (F, chunk, N, g, kw) in CONFIGS.items():
        if F <= 0:
            continue
        spec = P.VoxelGridSpec(g["origin"], g["dims"], g["resolution"])
        grid = O.Grid(spec.origin, spec.dims, spec.resolution)
        vox = {prec: P.Voxelizer(spec, P.VoxelizeConfig(precision=prec), 18, free_index=255)
               for prec in ("strict", "fast")}
        acc = {prec: {"frames": 0, "n_prims": N, "grid": list(g["dims"]), "pairs": 0,
                      "pairs_exact": True, "bins_exact": True, "worst_vo_rel": 0.0,
                      "n_vo_out_of_bound": 0, "worst_vc_rel": 0.0, "n_label_mismatch": 0,
                      "n_unexplained": 0, "n_resolvable": 0, "n_resolvable_mismatch": 0,
                      "voxels": 0, "oracle_s": 0.0} for prec in vox}
        for f0 in range(0, F, chunk):
            nf = min(chunk, F - f0)
            b = gen_frames(SEED, nf, N, 18, first_frame=f0, origin=spec.origin, dims=spec.dims,
                           resolution=spec.resolution, **kw)
            t0 = time.perf_counter()
            p = O.Prims.of(b)
            ref = O.voxelize(p, grid, O.Cfg(free_label=255))
            t_ref = time.perf_counter() - t0
            # the class sums' term magnitudes sum_i w_i |c_ik| (tests/parity.py)
            vc_abs = O.voxelize(O.Prims(p.mu, p.scale, p.rot, p.opacity, p.eps, np.abs(p.logits),
                                        p.n_valid), grid, O.Cfg(free_label=255))["v_c"]
            win = O.prep(O.Prims.of(b), grid, O.Cfg(free_label=255))
            off, ids = O.bins(win, grid.dims)
            C = ref["v_c"].shape[-1]
            for prec, vx in vox.items():
                cfg = vx.cfg
                r = vx(b, dense=True, bins=True)
                assert r.free_code == 255
                lab = r.labels.reshape(nf, -1).cpu().numpy()
                vo = r.v_o.reshape(nf, -1).cpu().numpy()
                vc = r.v_c.reshape(nf, -1, C).cpu().numpy()
                a = acc[prec]
                a["bins_exact"] &= bool(np.array_equal(r.bins["windows"].cpu().numpy(), win) and
                                        np.array_equal(r.bins["tile_off"].cpu().numpy(), off) and
                                        np.array_equal(r.bins["prim_ids"].cpu().numpy(), ids))
                a["pairs_exact"] &= int(r.n_pairs) == int(ref["n_pairs"])
                a["pairs"] += int(ref["n_pairs"])
                v = vo_check(vo, ref["v_o"], cfg.tau, prec)
                a["worst_vo_rel"] = max(a["worst_vo_rel"], v["worst_rel"])
                a["n_vo_out_of_bound"] += v["n_bad"]
                a["worst_vc_rel"] = max(a["worst_vc_rel"], vc_worst(vc, ref["v_c"], ref["v_o"],
                                                                    cfg.tau, vc_abs))
                lc = label_check(lab, ref["labels"], ref["v_o"], ref["v_c"], cfg.tau, r.free_code,
                                 vc_abs)
                a["n_label_mismatch"] += lc["n_mismatch"]
                a["n_unexplained"] += lc["n_unexplained"]
                a["n_resolvable"] += lc["n_resolvable"]
                a["n_resolvable_mismatch"] += round((1.0 - lc["agreement"]) * lc["n_resolvable"])
                a["voxels"] += int(lab.size)
                a["frames"] += nf
                a["oracle_s"] += t_ref
            del ref, vc_abs
        for prec, a in acc.items():
            a["label_agreement"] = 1.0 - a["n_resolvable_mismatch"] / max(a["n_resolvable"], 1)
            a["vc_limit"] = 2 * (VO_REL if prec == "strict" else VO_REL_TAIL)
            out["configs"][f"{name}_{prec}"] = a
            print(name, prec, json.dumps(a), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "parity_sweep.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    bad = [k for k, r in out["configs"].items()
           if not (r["bins_exact"] and r["pairs_exact"] and r["n_vo_out_of_bound"] == 0
                   and r["worst_vc_rel"] <= r["vc_limit"]
                   and r["n_unexplained"] == 0 and r["label_agreement"] >= 0.9999)]
    print("parity sweep", "FAILED: " + ", ".join(bad) if bad else "ok")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
