"""Parity criteria between the B200 path and the FP64 oracle (north_star):

* bins, windows, pair counts and confusion counts: bit-exact;
* densities:
    precision="strict" (default):
    |v_o - ref| <= 1e-5 * max(ref, floor)      1e-5 relative down to the floor,
    floor = max(1e-3*tau, 1e-5)                1e-3*tau, never
                                               below the default tau's 1e-5
                                               (tau = 0 has no tau scale);
    precision="fast":
    |v_o - ref| <= 3e-5 * max(ref, floor)      (the SFU log2 error, 2^-22.6
                                               absolute, and the once-rounded
                                               z steps are amplified by
                                               2/eps1 <= 10 in F and by F in
                                               exp(-F): F c (ln2 1.6e-7 +
                                               7e-8) reaches 2.4e-5 at the
                                               floor, F = 11.5, for c = 10;
                                               4,096 config-1 frames measured
                                               2.2e-5);
* class sums v_c: twice the v_o bound per mode, against the voxel's weight
  scale max(max_k T_k, max_k |v_c,k|, v_o, floor), T_k = sum_i w_i |c_ik|
  the term magnitude of class k (the oracle run with |logits|, ref["v_c_abs"],
  when the caller has it): every term w_i c_ik carries the relative error of
  w_i, so |dv_c,k| scales with T_k, and with mixed-sign logits cancelling
  inside v_c (and sigma < 1 under v_o) max(|v_c|, v_o) alone can be far
  below it;
* labels: a voxel may disagree only where the oracle's top-2 class scores
  differ by < LABEL_GAP * scale + 2 * CULL_DROP, scale being the voxel's
  weight scale of the v_c check (relative to the voxel's own term
  magnitude, no absolute floor of 1), or where the
  oracle's v_o lies within VO_REL of tau (a tau flip).  CULL_DROP is the
  block cull's per-voxel bound on the dropped mass: every
  class sum moves by < 2e-12, so a top-2 gap below twice that can flip.
  Overall agreement >= 99.99%, counted over the voxels whose oracle v_o
  exceeds CULL_DROP: below it every contribution may be culled (v_c = 0,
  label 0 at tau = 0, where the FP64 oracle takes the argmax of tail
  values); those voxels still have to satisfy the near-tie rule above.
"""
from __future__ import annotations

import numpy as np

VO_REL = 1e-5                # strict
VO_REL_TAIL = 3e-5           # fast
VO_TAIL_FLOOR_FRAC_TAU = 1e-3
VO_MIN_FLOOR = 1e-5          # = 1e-3 * the default tau (0.01)
LABEL_GAP = 1e-5
CULL_DROP = 2e-12            # kDropBound, csrc/sqv_common.cuh
MIN_AGREEMENT = 0.9999


def vo_check(gpu, ref, tau, mode="strict"):
    gpu = np.asarray(gpu, np.float64).ravel()
    ref = np.asarray(ref, np.float64).ravel()
    err = np.abs(gpu - ref)
    out = {}
    bad = np.zeros(err.shape, bool)
    tail_floor = max(VO_TAIL_FLOOR_FRAC_TAU * tau, VO_MIN_FLOOR)
    tiers = ((("tier1", VO_REL, tail_floor),) if mode == "strict" else
             (("tier1", VO_REL_TAIL, tail_floor),))
    for name, rel, floor in tiers:
        scaled = err / np.maximum(ref, floor)
        out[f"worst_rel_{name}"] = float(scaled.max()) if err.size else 0.0
        bad |= scaled > rel
    out["worst_rel"] = out["worst_rel_tier1"]
    out["n_bad"] = int(bad.sum())
    out["bad_idx"] = np.flatnonzero(bad)[:10]
    return out


def weight_scale(ref_vo, ref_vc, tau, ref_vc_abs=None):
    """Per voxel: max(max_k T_k, max_k |v_c,k|, v_o, floor) (see above)."""
    C = ref_vc.shape[-1]
    vc = np.abs(np.asarray(ref_vc, np.float64)).reshape(-1, C).max(axis=-1)
    vo = np.asarray(ref_vo, np.float64).ravel()
    floor = max(VO_TAIL_FLOOR_FRAC_TAU * tau, VO_MIN_FLOOR)
    s = np.maximum(np.maximum(vc, vo), floor)
    if ref_vc_abs is not None:
        s = np.maximum(s, np.asarray(ref_vc_abs, np.float64).reshape(-1, C).max(axis=-1))
    return s


def label_check(gpu_lab, ref_lab, ref_vo, ref_vc, tau, free_code, ref_vc_abs=None):
    g = np.asarray(gpu_lab).ravel()
    r = np.asarray(ref_lab).ravel()
    vo = np.asarray(ref_vo, np.float64).ravel()
    C = ref_vc.shape[-1]
    vc = np.asarray(ref_vc, np.float64).reshape(-1, C)
    wscale = weight_scale(ref_vo, ref_vc, tau, ref_vc_abs)
    mism = np.flatnonzero(g != r)
    unexplained = []
    for v in mism:
        if abs(vo[v] - tau) <= VO_REL * max(tau, 1e-30):
            continue  # tau flip
        if g[v] != free_code and r[v] != free_code:
            top = vc[v, r[v]]
            if top - vc[v, g[v]] <= LABEL_GAP * wscale[v] + 2 * CULL_DROP:
                continue  # near-tie in the oracle's scores
        unexplained.append(int(v))
    resolvable = vo > CULL_DROP
    n_res = int(resolvable.sum())
    agree = 1.0 - int((g != r)[resolvable].sum()) / max(n_res, 1)
    return {"n_mismatch": int(mism.size), "unexplained": unexplained[:10],
            "n_unexplained": len(unexplained), "agreement": agree,
            "agreement_all": 1.0 - mism.size / max(g.size, 1), "n_resolvable": n_res}


def assert_parity(gpu, ref, tau, free_code, check_vc=True, mode="strict",
                  min_agreement=MIN_AGREEMENT):
    """gpu/ref: dicts with v_o [F,V], v_c [F,V,C] (ref FP64), labels [F,V]."""
    vo = vo_check(gpu["v_o"], ref["v_o"], tau, mode)
    assert vo["n_bad"] == 0, f"v_o out of tolerance: {vo}"
    vc_abs = ref.get("v_c_abs")
    lab = label_check(gpu["labels"], ref["labels"], ref["v_o"], ref["v_c"], tau, free_code,
                      vc_abs)
    assert lab["n_unexplained"] == 0, f"unexplained label mismatches: {lab}"
    assert lab["agreement"] >= min_agreement, lab
    if check_vc:
        # class sums against the voxel's weight scale (the term magnitude
        # when ref carries v_c_abs); twice the v_o bound: the B operand's
        # 3xTF32 split and the class weights' own rounding add to w's error
        vc_g = np.asarray(gpu["v_c"], np.float64)
        vc_r = np.asarray(ref["v_c"], np.float64)
        scale = weight_scale(ref["v_o"], vc_r, tau, vc_abs).reshape(vc_r.shape[:-1] + (1,))
        rel = np.abs(vc_g - vc_r) / scale
        lim = 2 * (VO_REL if mode == "strict" else VO_REL_TAIL)
        assert float(rel.max(initial=0.0)) <= lim, f"v_c worst {float(rel.max())}"
    return vo, lab
