"""Diagnostics (GPU): FP32/SFU error of F and exp(-F) vs the FP64 oracle,
binned by the exponent amplification 2/eps1, and the v_o error profile of a
config-1 frame binned by v_o.  Writes gpurun_out/diag_precision.json."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import oracle as O  # noqa: E402
import paper_2511_17361_b200 as P  # noqa: E402
from paper_2511_17361_b200.density import density_pairs  # noqa: E402
from paper_2511_17361_b200.scenegen import gen_frames  # noqa: E402


def pairs_error():
    rng = np.random.default_rng(3)
    n, per = 4000, 64
    b = gen_frames(5, 1, n, 2, origin=(-5, -5, -5), dims=(25, 25, 25), resolution=0.4,
                   smin=0.2, smax=2.0)
    sc = np.asarray(b.scale)[0]
    d = rng.normal(size=(n, per, 3))
    d /= np.linalg.norm(d, axis=-1, keepdims=True)
    r = rng.uniform(0.05, 4.0, size=(n, per, 1))
    R = P.quat_to_matrix(np.asarray(b.rot)[0])          # local->world
    xl = d * r * sc[:, None, :]
    xw = np.einsum("nij,npj->npi", R, xl) + np.asarray(b.mu)[0][:, None, :]
    pp = np.repeat(np.arange(n), per).astype(np.int32)
    F, dens = density_pairs(b, xw.reshape(-1, 3), pp)
    Fr, dr = O.density(O.Prims.of(b), xw.reshape(-1, 3), pp)
    e1 = np.clip(np.asarray(b.eps)[0, :, 0], 0.2, 2.0)
    amp = np.repeat(2.0 / e1, per)
    out = {}
    live = (Fr > 1e-3) & (Fr < 80)
    relF = np.abs(F.astype(np.float64) - Fr) / Fr
    for lo, hi in [(1, 2), (2, 4), (4, 7), (7, 10.01)]:
        m = live & (amp >= lo) & (amp < hi)
        out[f"amp_{lo}_{hi}"] = {"n": int(m.sum()), "relF_max": float(relF[m].max()),
                                 "relF_p99": float(np.quantile(relF[m], 0.99)),
                                 "relF_over_amp_max": float((relF[m] / amp[m]).max())}
    big = dr > 1e-6
    out["density_rel_over_F_max"] = float((np.abs(dens[big] - dr[big]) / dr[big] /
                                           np.maximum(Fr[big], 1e-3)).max())
    return out


def vo_profile(seed=11, n=256):
    spec, cfg = P.VoxelGridSpec(), P.VoxelizeConfig()
    b = gen_frames(seed, 1, n, 18)
    r = P.Voxelizer(spec, cfg, 18)(b)
    vo = r.v_o.reshape(-1).cpu().numpy().astype(np.float64)
    ref = O.voxelize(O.Prims.of(b), O.Grid(), O.Cfg(free_label=18))["v_o"][0]
    rel = np.abs(vo - ref) / np.maximum(ref, 1e-300)
    out = {}
    for lo, hi in [(1e-6, 1e-5), (1e-5, 1e-4), (1e-4, 1e-3), (1e-3, 1e-2), (1e-2, 1e-1),
                   (1e-1, 1e9)]:
        m = (ref >= lo) & (ref < hi)
        if m.any():
            out[f"vo_{lo:g}_{hi:g}"] = {"n": int(m.sum()), "rel_max": float(rel[m].max()),
                                        "rel_p999": float(np.quantile(rel[m], 0.999)),
                                        "n_over_1e-5": int((rel[m] > 1e-5).sum())}
    return out


if __name__ == "__main__":
    res = {"pairs": pairs_error(), "vo_config1": vo_profile(),
           "vo_config2_frame": vo_profile(7, 2000)}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "diag_precision.json"), "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1))
