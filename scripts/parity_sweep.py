"""Parity at the benchmark's sizes over many frames (GPU box): the bench
configs' own generator (scenegen.gen_frames, the bench seed) voxelized by
the product path in both precisions, every frame checked in full against the
FP64 oracle (oracle/, the checker): bins and pair counts exact, the worst
|dv_o| / max(v_o, floor), label agreement and unexplained mismatches
(tests/parity.py rules).  Writes gpurun_out/parity_sweep.json.

usage: python scripts/parity_sweep.py [frames_c2] [frames_c3] [frames_c1]
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
from parity import label_check, vo_check  # noqa: E402

SEED = 20251117  # bench.py default
CONFIGS = {  # name: (frames, n_prims, gen kwargs)
    "config2": (int(sys.argv[1]) if len(sys.argv) > 1 else 16, 2000, {}),
    "config3": (int(sys.argv[2]) if len(sys.argv) > 2 else 4, 4000, {"emin": 0.1}),
    "config1": (int(sys.argv[3]) if len(sys.argv) > 3 else 16, 256, {}),
}


def main():
    spec = P.VoxelGridSpec()
    grid = O.Grid(spec.origin, spec.dims, spec.resolution)
    out = {"oracle_threads": O.threads(), "configs": {}}
    for name, (F, N, kw) in CONFIGS.items():
        b = gen_frames(SEED, F, N, 18, **kw)
        t0 = time.perf_counter()
        ref = O.voxelize(O.Prims.of(b), grid, O.Cfg(free_label=255))
        t_ref = time.perf_counter() - t0
        win = O.prep(O.Prims.of(b), grid, O.Cfg(free_label=255))
        off, ids = O.bins(win, grid.dims)
        for prec in ("strict", "fast"):
            cfg = P.VoxelizeConfig(precision=prec)
            vox = P.Voxelizer(spec, cfg, 18, free_index=255)
            r = vox(b, dense=True, bins=True)
            assert r.free_code == 255
            lab = r.labels.reshape(F, -1).cpu().numpy()
            vo = r.v_o.reshape(F, -1).cpu().numpy()
            bins_exact = (np.array_equal(r.bins["windows"].cpu().numpy(), win) and
                          np.array_equal(r.bins["tile_off"].cpu().numpy(), off) and
                          np.array_equal(r.bins["prim_ids"].cpu().numpy(), ids))
            v = vo_check(vo, ref["v_o"], cfg.tau, prec)
            lc = label_check(lab, ref["labels"], ref["v_o"], ref["v_c"], cfg.tau, r.free_code)
            rec = {"frames": F, "n_prims": N, "pairs": int(ref["n_pairs"]),
                   "pairs_exact": int(r.n_pairs) == int(ref["n_pairs"]), "bins_exact": bins_exact,
                   "worst_vo_rel": v["worst_rel"], "n_vo_out_of_bound": v["n_bad"],
                   "label_agreement": lc["agreement"], "n_label_mismatch": lc["n_mismatch"],
                   "n_unexplained": lc["n_unexplained"], "voxels": int(lab.size),
                   "oracle_s": t_ref}
            out["configs"][f"{name}_{prec}"] = rec
            print(name, prec, json.dumps(rec), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "parity_sweep.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    bad = [k for k, r in out["configs"].items()
           if not (r["bins_exact"] and r["pairs_exact"] and r["n_vo_out_of_bound"] == 0
                   and r["n_unexplained"] == 0 and r["label_agreement"] >= 0.9999)]
    print("parity sweep", "FAILED: " + ", ".join(bad) if bad else "ok")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
