"""B200 path vs the FP64 oracle / the reference's golden vectors (-m gpu).

Every call goes through libsqv.so (include/sqv.h) via the package's public
API; the oracle (oracle/) is only the checker.
"""
import glob
import os
import re

import numpy as np
import pytest

from conftest import GOLDEN, load_golden
from oracle import oracle as O
from parity import assert_parity, label_check, vo_check

pytestmark = pytest.mark.gpu


def _pkg():
    import paper_2511_17361_b200 as P
    return P


def _batch_from(g):
    P = _pkg()
    return P.PrimitiveBatch(*(np.asarray(g[k])[None] for k in
                              ("mu", "scale", "rot", "opacity", "eps", "logits")))


def _run(batch, spec, cfg, C, free=None, truncate=True, bins=False):
    P = _pkg()
    vox = P.Voxelizer(spec, cfg, C, free, truncate=truncate)
    r = vox(batch, dense=True, bins=bins)
    F = batch.n_frames
    out = {"labels": r.labels.reshape(F, -1).cpu().numpy(),
           "v_o": r.v_o.reshape(F, -1).cpu().numpy(),
           "v_c": r.v_c.reshape(F, spec.n_voxels, C).cpu().numpy(),
           "n_pairs": r.n_pairs, "free_code": r.free_code}
    if bins:
        out["windows"] = r.bins["windows"].cpu().numpy()
        out["tile_off"] = r.bins["tile_off"].cpu().numpy()
        out["prim_ids"] = r.bins["prim_ids"].cpu().numpy()
    return out


def _oracle(batch, spec, cfg, free_code, truncate=True):
    p = O.Prims.of(batch)
    grid = O.Grid(spec.origin, spec.dims, spec.resolution)
    c = O.Cfg(cfg.tau, cfg.neighborhood_radius, truncate, cfg.semantic_mode == "prob-sum",
              free_code, cfg.window_extent)
    r = O.voxelize(p, grid, c)
    r["windows"] = O.prep(p, grid, c)
    if cfg.semantic_mode == "logit-sum":
        # the class sums' term magnitudes sum_i w_i |c_ik| (parity.weight_scale)
        pa = O.Prims(p.mu, p.scale, p.rot, p.opacity, p.eps, np.abs(p.logits), p.n_valid)
        r["v_c_abs"] = O.voxelize(pa, grid, c)["v_c"]
    return r, grid


# ---- point-wise math vs the reference's sqocc.core ------------------------

def test_density_pairs_vs_reference_core():
    from paper_2511_17361_b200.density import density_pairs
    g = load_golden("core_pairs.npz")
    F, d = density_pairs(_batch_from(g), g["points"], g["pair_prim"])
    Fr, dr = g["F"], g["density"]
    live = Fr < 80
    relF = np.abs(F[live] - Fr[live]) / np.maximum(Fr[live], 1e-3)
    assert relF.max() < 2e-5, relF.max()
    # exp(-F): error ~ |dF|; relative 1e-5 where the density is >= 1e-3
    big = dr >= 1e-3
    assert np.max(np.abs(d[big] - dr[big]) / dr[big]) < 1e-5
    assert np.all(np.abs(d - dr) <= 1e-5 * np.maximum(dr, 1e-3) + 1e-38)


# ---- reference golden scenes ------------------------------------------------

@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "voxelize_*.npz"))),
                         ids=lambda p: os.path.basename(p)[9:-4])
def test_golden_scenes(path):
    P = _pkg()
    g = dict(np.load(path))
    C = g["logits"].shape[1]
    spec = P.VoxelGridSpec(tuple(g["origin"]), tuple(int(x) for x in g["dims"]), float(g["res"]))
    cfg = P.VoxelizeConfig(float(g["tau"]), int(g["radius"]),
                           "prob-sum" if bool(g["prob_sum"]) else "logit-sum")
    out = _run(_batch_from(g), spec, cfg, C, int(g["free_label"]), truncate=bool(g["truncate"]),
               bins=True)
    np.testing.assert_array_equal(out["windows"][0], g["windows"])
    np.testing.assert_array_equal(out["tile_off"], g["tile_off"])
    np.testing.assert_array_equal(out["prim_ids"], g["prim_ids"])
    assert out["n_pairs"] == int(g["n_pairs"])
    ref = {"v_o": g["v_o"][None], "v_c": g["v_c"][None], "labels": g["labels"][None]}
    assert_parity(out, ref, float(g["tau"]), int(g["free_label"]))


# ---- seeded scenes vs the oracle ----------------------------------------------

def _scene(seed, n, C=18, **kw):
    from paper_2511_17361_b200.scenegen import gen_frames
    return gen_frames(seed, kw.pop("frames", 1), n, C, **kw)


def test_config1_occ3d_256():
    """Config 1: 256 SQs on the Occ3D grid, full parity + exact bins."""
    P = _pkg()
    spec, cfg = P.VoxelGridSpec(), P.VoxelizeConfig()
    b = _scene(11, 256)
    out = _run(b, spec, cfg, 18, bins=True)
    ref, grid = _oracle(b, spec, cfg, out["free_code"])
    np.testing.assert_array_equal(out["windows"], ref["windows"])
    off, ids = O.bins(ref["windows"], grid.dims)
    np.testing.assert_array_equal(out["tile_off"], off)
    np.testing.assert_array_equal(out["prim_ids"], ids)
    assert out["n_pairs"] == ref["n_pairs"]
    vo, lab = assert_parity(out, ref, cfg.tau, out["free_code"])
    print("config1 worst v_o rel", vo["worst_rel"], "label agreement", lab["agreement"])


def test_fast_precision_mode():
    """precision="fast" (all logs on the SFU): labels unchanged, densities within
    3e-5 relative down to 1e-3*tau."""
    P = _pkg()
    spec, cfg = P.VoxelGridSpec(), P.VoxelizeConfig(precision="fast")
    b = _scene(11, 256)
    out = _run(b, spec, cfg, 18)
    ref, _ = _oracle(b, spec, cfg, out["free_code"])
    assert_parity(out, ref, cfg.tau, out["free_code"], mode="fast")


@pytest.mark.parametrize("seed", range(20))
def test_acceptance4_bruteforce_equivalence(seed):
    """SPEC.md:630 #4: <=50 prims, 32^3: untruncated voxelize == bruteforce oracle."""
    P = _pkg()
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 51))
    spec = P.VoxelGridSpec((-6.4, -6.4, -6.4), (32, 32, 32), 0.4)
    cfg = P.VoxelizeConfig()
    b = _scene(500 + seed, n, C=8, origin=spec.origin, dims=spec.dims,
               resolution=spec.resolution, smax=2.0)
    out = _run(b, spec, cfg, 8, truncate=False)
    ref, _ = _oracle(b, spec, cfg, out["free_code"], truncate=False)
    assert out["n_pairs"] == ref["n_pairs"]
    assert_parity(out, ref, cfg.tau, out["free_code"])
    # default N=5 window: parity with the truncated oracle, and truncation
    # soundness: every voxel whose label differs from the
    # brute-force label lost positive tail mass.
    tr = _run(b, spec, cfg, 8, truncate=True)
    tref, _ = _oracle(b, spec, cfg, out["free_code"], truncate=True)
    assert_parity(tr, tref, cfg.tau, out["free_code"])
    diff = tref["labels"] != ref["labels"]
    omitted = ref["v_o"] - tref["v_o"]
    assert np.all(omitted[diff] > 0)
    assert np.all(omitted >= -1e-12 * np.maximum(ref["v_o"], 1e-30))


@pytest.mark.parametrize("kw", [dict(emin=0.1), dict(smax=1.0), dict(smin=0.05, smax=0.6)],
                         ids=["stress_eps", "sparse", "needles"])
def test_stress_sets(kw):
    P = _pkg()
    spec, cfg = P.VoxelGridSpec(), P.VoxelizeConfig()
    b = _scene(21, 600, **kw)
    out = _run(b, spec, cfg, 18)
    ref, _ = _oracle(b, spec, cfg, out["free_code"])
    assert_parity(out, ref, cfg.tau, out["free_code"])


def test_prob_sum_and_ragged_batch_determinism():
    """prob-sum mode; ragged frames (n_valid); a frame's output does not depend
    on its batch position (bit-identical)."""
    P = _pkg()
    spec = P.VoxelGridSpec((-8.0, -8.0, -2.0), (40, 40, 16), 0.4)
    cfg = P.VoxelizeConfig(semantic_mode="prob-sum")
    b = _scene(31, 120, C=5, frames=3, origin=spec.origin, dims=spec.dims, smax=2.0)
    b.n_valid = np.array([120, 37, 0], np.int32)
    out = _run(b, spec, cfg, 5)
    ref, _ = _oracle(b, spec, cfg, out["free_code"])
    assert_parity(out, ref, cfg.tau, out["free_code"])
    assert np.all(out["labels"][2] == out["free_code"]) and np.all(out["v_o"][2] == 0)
    single = _run(b.frames(1, 2), spec, cfg, 5)
    assert np.array_equal(single["v_o"][0], out["v_o"][1])
    assert np.array_equal(single["v_c"][0], out["v_c"][1])
    again = _run(b, spec, cfg, 5)
    assert all(np.array_equal(again[k], out[k]) for k in ("labels", "v_o", "v_c"))


def test_config2_frame_large_properties():
    """One config-2 frame (2k SQs): bins exact, pair count exact, >= 99.99% label
    agreement, v_o within tolerance."""
    P = _pkg()
    spec, cfg = P.VoxelGridSpec(), P.VoxelizeConfig()
    b = _scene(7, 2000)
    out = _run(b, spec, cfg, 18, bins=True)
    ref, grid = _oracle(b, spec, cfg, out["free_code"])
    np.testing.assert_array_equal(out["windows"], ref["windows"])
    off, ids = O.bins(ref["windows"], grid.dims)
    np.testing.assert_array_equal(out["tile_off"], off)
    np.testing.assert_array_equal(out["prim_ids"], ids)
    assert out["n_pairs"] == ref["n_pairs"]
    vo, lab = assert_parity(out, ref, cfg.tau, out["free_code"])
    print("config2 pairs", ref["n_pairs"], "worst v_o rel", vo["worst_rel"], "agreement",
          lab["agreement"])


def test_fine_grid_config4_slice():
    """Config 4 geometry (400x400x32 @0.2) with a reduced primitive count."""
    P = _pkg()
    spec = P.VoxelGridSpec((-40.0, -40.0, -1.0), (400, 400, 32), 0.2)
    cfg = P.VoxelizeConfig()
    b = _scene(9, 300, origin=spec.origin, dims=spec.dims, resolution=spec.resolution)
    out = _run(b, spec, cfg, 18, bins=True)
    ref, grid = _oracle(b, spec, cfg, out["free_code"])
    off, ids = O.bins(ref["windows"], grid.dims)
    np.testing.assert_array_equal(out["tile_off"], off)
    np.testing.assert_array_equal(out["prim_ids"], ids)
    assert_parity(out, ref, cfg.tau, out["free_code"])


@pytest.mark.parametrize("which", ["config3", "config4"])
def test_full_frame_configs_3_and_4(which):
    """One full frame of config 3 (4k SQs, eps in [0.1, 2]: near-cuboids and
    needles, clamped per core.py:162-165) and of config 4 (8k SQs on
    400x400x32 @0.2 m, ~1.8 G pairs): bins, pair count, densities and labels
    against the FP64 oracle at the BASELINE sizes."""
    P = _pkg()
    if which == "config3":
        spec = P.VoxelGridSpec()
        b = _scene(21, 4000, emin=0.1)
    else:
        spec = P.VoxelGridSpec((-40.0, -40.0, -1.0), (400, 400, 32), 0.2)
        b = _scene(22, 8000, origin=spec.origin, dims=spec.dims, resolution=spec.resolution)
    cfg = P.VoxelizeConfig()
    out = _run(b, spec, cfg, 18, bins=True)
    ref, grid = _oracle(b, spec, cfg, out["free_code"])
    np.testing.assert_array_equal(out["windows"], ref["windows"])
    off, ids = O.bins(ref["windows"], grid.dims)
    np.testing.assert_array_equal(out["tile_off"], off)
    np.testing.assert_array_equal(out["prim_ids"], ids)
    assert out["n_pairs"] == ref["n_pairs"]
    vo, lab = assert_parity(out, ref, cfg.tau, out["free_code"])
    print(which, "pairs", ref["n_pairs"], "worst v_o rel", vo["worst_rel"], "agreement",
          lab["agreement"])


# ---- drop-in API ----------------------------------------------------------------

def test_dropin_scene_api_and_spec_examples():
    P = _pkg()
    classes = P.ClassTable(("a",))
    spec = P.VoxelGridSpec((-2.0, -2.0, -2.0), (8, 8, 8), 0.5)
    # SPEC.md:351 empty scene -> all free, v_o == 0
    sem, dense = P.voxelize(P.Scene([], classes), spec)
    assert np.all(sem.labels == classes.free_index) and np.all(dense.v_o == 0)
    # SPEC.md:352 unit sphere on a voxel centre, C=1 -> v_o = 1 there, class 0
    sq = P.SuperQuadric(mu=[0.25, 0.25, 0.25], scale=[1, 1, 1], rot=[1, 0, 0, 0], opacity=1.0,
                        logits=[0.3], eps1=1.0, eps2=1.0)
    sem, dense = P.voxelize(P.Scene([sq], classes), spec)
    assert dense.v_o.shape == (8, 8, 8) and dense.v_c.shape == (8, 8, 8, 1)
    assert abs(dense.v_o[4, 4, 4] - 1.0) < 1e-6 and sem.labels[4, 4, 4] == 0
    # finalize: tau = 0 -> no free voxel where anything contributed; tau = inf -> all free
    assert np.all(P.finalize(dense, 0.0, classes).labels[dense.v_o > 0] == 0)
    assert np.all(P.finalize(dense, float("inf"), classes).labels == classes.free_index)
    # tau sweep monotonicity
    occ = [int(np.sum(P.finalize(dense, t, classes).labels != classes.free_index))
           for t in (0.005, 0.01, 0.02)]
    assert occ[0] >= occ[1] >= occ[2]
    # finalize keeps the grid geometry: from dense.spec, or spec=; a bare
    # non-default DenseGrids is rejected rather than given the Occ3D origin
    assert P.finalize(dense, 0.01, classes).spec == spec
    bare = P.DenseGrids(dense.v_o, dense.v_c)
    with pytest.raises(ValueError, match="spec="):
        P.finalize(bare, 0.01, classes)
    np.testing.assert_array_equal(P.finalize(bare, 0.01, classes, spec=spec).labels, sem.labels)


def test_sigma_scaling_argmax_invariance():
    """scaling all sigma leaves labels unchanged where occupied."""
    P = _pkg()
    spec, cfg = P.VoxelGridSpec(), P.VoxelizeConfig()
    b = _scene(41, 300, smax=1.5)
    b2 = P.PrimitiveBatch(b.mu, b.scale, b.rot, b.opacity * 0.5, b.eps, b.logits)
    o1 = _run(b, spec, cfg, 18)
    o2 = _run(b2, spec, cfg, 18)
    both = (o1["labels"] != o1["free_code"]) & (o2["labels"] != o2["free_code"])
    assert np.mean(o1["labels"][both] == o2["labels"][both]) > 0.9999


def test_invalid_primitive_messages():
    P = _pkg()
    spec = P.VoxelGridSpec((-2.0, -2.0, -2.0), (8, 8, 8), 0.5)
    vox = P.Voxelizer(spec, P.VoxelizeConfig(), 2)
    base = _scene(3, 4, C=2, origin=spec.origin, dims=spec.dims, resolution=spec.resolution)
    cases = [("scale", (0, 1, 2), -1.0, "scale components must be strictly positive"),
             ("opacity", (0, 2), 1.5, "opacity must lie in [0, 1]"),
             ("mu", (0, 3, 0), np.nan, "mu/scale must be finite"),
             ("logits", (0, 0, 1), np.inf, "logits must be finite")]
    for field, idx, val, msg in cases:
        arrs = {k: np.array(getattr(base, k)) for k in P.PrimitiveBatch.FIELDS}
        arrs[field][idx] = val
        with pytest.raises(ValueError, match=re.escape(msg)):
            vox(P.PrimitiveBatch(**arrs))
    arrs = {k: np.array(getattr(base, k)) for k in P.PrimitiveBatch.FIELDS}
    arrs["rot"][0, 1] = 0.0
    with pytest.raises(ValueError, match="near-zero quaternion"):
        vox(P.PrimitiveBatch(**arrs))


# ---- metrics ---------------------------------------------------------------------

def test_confusion_kernel_vs_golden():
    from paper_2511_17361_b200.metrics import confusion_matrix
    g = load_golden("confusion.npz")
    s = c0 = 0
    for n, C in zip(g["lens"], g["C"]):
        k = (C + 1) ** 2
        cm = confusion_matrix(g["pred"][s:s + n], g["gt"][s:s + n], int(C)).cpu().numpy()
        np.testing.assert_array_equal(cm.ravel(), g["cm"][c0:c0 + k])
        s += n
        c0 += k


def test_confusion_large_and_iou_examples():
    P = _pkg()
    from paper_2511_17361_b200 import metrics as M
    rng = np.random.default_rng(5)
    a = rng.integers(0, 19, size=3_000_017).astype(np.uint8)
    b = np.where(rng.uniform(size=a.size) < 0.7, a, rng.integers(0, 19, size=a.size)).astype(np.uint8)
    a[a == 18] = 255
    cm = M.confusion_matrix(a, b, 18).cpu().numpy()
    np.testing.assert_array_equal(cm, O.confusion(a, b, 18))
    # 2x2x1, pred {(0,0),(1,0)}, gt {(1,0),(1,1)} -> 1/3
    classes = P.ClassTable(("x",))
    spec = P.VoxelGridSpec(dims=(2, 2, 1))
    pl = np.full((2, 2, 1), 1)
    gl = np.full((2, 2, 1), 1)
    pl[0, 0, 0] = pl[1, 0, 0] = 0
    gl[1, 0, 0] = gl[1, 1, 0] = 0
    pred = P.SemanticGrid(pl, spec, classes)
    gt = P.SemanticGrid(gl, spec, classes)
    assert abs(M.voxel_iou(pred, gt) - 1 / 3) < 1e-12
    assert M.voxel_iou(pred, pred) == 1.0
    per, m = M.miou(pred, pred)
    assert m == 1.0


def test_stream_api_matches_direct_calls():
    """Voxelizer.stream (overlapped copies) gives the same labels as direct calls."""
    import torch
    P = _pkg()
    spec = P.VoxelGridSpec((-8.0, -8.0, -2.0), (40, 40, 16), 0.4)
    vox = P.Voxelizer(spec, P.VoxelizeConfig(), 6)
    batches = [_scene(60 + k, 150, C=6, frames=3, origin=spec.origin, dims=spec.dims, smax=2.0)
               for k in range(4)]
    pinned = [P.PrimitiveBatch(**{f: torch.from_numpy(np.asarray(getattr(b, f))).pin_memory()
                                  for f in P.PrimitiveBatch.FIELDS}) for b in batches]
    seen = []
    labels = vox.stream(pinned, on_device=lambda k, r: seen.append(k))
    assert seen == [0, 1, 2, 3]
    for b, lab in zip(batches, labels):
        direct = vox(b).labels.cpu()
        assert torch.equal(direct, lab)


@pytest.mark.parametrize("nb,ragged", [(1, False), (2, False), (4, False), (4, True)])
def test_stream_edge_ranges_match_direct_calls(nb, ragged, monkeypatch):
    """Voxelizer.stream splits its first and last batch into frame ranges
    (pipeline fill/drain) and triple-buffers inputs and labels: labels, v_o,
    v_c and the pair counts handed to on_device equal one direct call per
    batch, bit for bit.  The evaluator kernel is pinned (SQV_STREAM=1): its
    automatic choice depends on the batch's density and tile count, and the
    chunk-staged and streaming kernels agree to rounding, not bit for bit."""
    import torch
    monkeypatch.setenv("SQV_STREAM", "1")
    P = _pkg()
    spec = P.VoxelGridSpec((-8.0, -8.0, -2.0), (40, 40, 16), 0.4)
    vox = P.Voxelizer(spec, P.VoxelizeConfig(), 6)
    F = 40
    batches = []
    for k in range(nb):
        b = _scene(90 + k, 150, C=6, frames=F, origin=spec.origin, dims=spec.dims, smax=2.0)
        if ragged:
            b = P.PrimitiveBatch(b.mu, b.scale, b.rot, b.opacity, b.eps, b.logits,
                                 n_valid=np.random.default_rng(k).integers(0, 151, F)
                                 .astype(np.int32))
        batches.append(b)
    pinned = [P.PrimitiveBatch(**{f: torch.from_numpy(np.asarray(getattr(b, f))).pin_memory()
                                  for f in P.PrimitiveBatch.FIELDS}, n_valid=b.n_valid)
              for b in batches]
    got = {}

    def cb(k, r):
        got[k] = (r.v_o.clone(), r.v_c.clone(), r.n_pairs, r.n_entries)

    labels = vox.stream(pinned, on_device=cb, edge_pieces=4)
    torch.cuda.synchronize()
    assert sorted(got) == list(range(nb))
    for k, (b, lab) in enumerate(zip(batches, labels)):
        d = vox(b)
        assert torch.equal(d.labels.cpu(), lab)
        assert torch.equal(d.v_o, got[k][0]) and torch.equal(d.v_c, got[k][1])
        assert (d.n_pairs, d.n_entries) == got[k][2:]


def test_stream_error_leaves_the_voxelizer_usable():
    """An invalid primitive in the middle of a stream raises the package's
    ValueError (after every stream of the call is drained), and the same
    Voxelizer streams correctly afterwards."""
    import torch
    P = _pkg()
    spec = P.VoxelGridSpec((-8.0, -8.0, -2.0), (40, 40, 16), 0.4)
    vox = P.Voxelizer(spec, P.VoxelizeConfig(), 6)
    batches = [_scene(120 + k, 150, C=6, frames=16, origin=spec.origin, dims=spec.dims, smax=2.0)
               for k in range(4)]
    bad_scale = np.array(batches[2].scale, copy=True)
    bad_scale[13, 7, 1] = -1.0
    bad = P.PrimitiveBatch(batches[2].mu, bad_scale, batches[2].rot, batches[2].opacity,
                           batches[2].eps, batches[2].logits)
    pin = lambda b: P.PrimitiveBatch(**{f: torch.from_numpy(np.asarray(getattr(b, f)))
                                         .pin_memory() for f in P.PrimitiveBatch.FIELDS})
    # a middle batch (one call) and the last one (run as frame ranges): the
    # frame index is the batch's either way
    with pytest.raises(ValueError, match="frame 13 primitive 7"):
        vox.stream([pin(b) for b in batches[:2]] + [pin(bad), pin(batches[3])])
    with pytest.raises(ValueError, match="frame 13 primitive 7"):
        vox.stream([pin(b) for b in batches[:2]] + [pin(bad)])
    labels = vox.stream([pin(b) for b in batches])
    for b, lab in zip(batches, labels):
        assert torch.equal(vox(b).labels.cpu(), lab)


def test_truncation_report_soundness():
    """cmd_voxelize --oracle: omitted mass is non-negative,
    every label flip lost mass, and the omitted mass stays under the summed
    per-primitive tail bound."""
    P = _pkg()
    from paper_2511_17361_b200.voxelize import truncation_report
    spec = P.VoxelGridSpec((-6.4, -6.4, -6.4), (32, 32, 32), 0.4)
    b = _scene(77, 40, C=8, origin=spec.origin, dims=spec.dims, resolution=spec.resolution,
               smax=1.5)
    rep = truncation_report(b, spec, P.VoxelizeConfig())
    assert rep["sound"]
    assert rep["min_dvo"] >= -1e-6
    assert rep["max_omitted_mass"] <= rep["sum_tail_bound"] * (1 + 1e-4) + 1e-6
    print(rep)


@pytest.mark.parametrize("C", [1, 3, 24, 32])
def test_class_counts(C):
    """Every evaluator instantiation: C <= 24 runs on tcgen05, C = 32 on the
    CUDA-core evaluator (sigma does not fit the N = 32 tensor-core tile)."""
    P = _pkg()
    spec = P.VoxelGridSpec((-8.0, -8.0, -2.0), (40, 40, 16), 0.4)
    cfg = P.VoxelizeConfig()
    b = _scene(90 + C, 150, C=C, origin=spec.origin, dims=spec.dims, smax=2.0)
    out = _run(b, spec, cfg, C)
    ref, _ = _oracle(b, spec, cfg, out["free_code"])
    assert_parity(out, ref, cfg.tau, out["free_code"])


def test_ffma_and_tensor_core_evaluators_agree(monkeypatch):
    """SQV_EVAL=ffma (CUDA-core accumulation) vs the default tcgen05 path."""
    P = _pkg()
    spec, cfg = P.VoxelGridSpec(), P.VoxelizeConfig()
    b = _scene(13, 400)
    tc_out = _run(b, spec, cfg, 18)
    monkeypatch.setenv("SQV_EVAL", "ffma")
    ff_out = _run(b, spec, cfg, 18)
    assert np.mean(tc_out["labels"] == ff_out["labels"]) > 0.99999
    # 3xTF32 products (~2^-21 relative each) vs FP32 FFMA (2^-24)
    np.testing.assert_allclose(tc_out["v_o"], ff_out["v_o"], rtol=5e-6, atol=1e-9)


def test_degenerate_inputs_and_free_index():
    """N = 0 primitives, tau = inf, and a free_index outside a byte."""
    P = _pkg()
    spec = P.VoxelGridSpec((-2.0, -2.0, -2.0), (9, 7, 5), 0.5)
    z = lambda *s: np.zeros(s)
    empty = P.PrimitiveBatch(z(2, 0, 3), z(2, 0, 3), z(2, 0, 4), z(2, 0), z(2, 0, 2), z(2, 0, 3))
    r = P.Voxelizer(spec, P.VoxelizeConfig(), 3)(empty)
    assert r.n_pairs == 0 and bool((r.labels == r.free_code).all()) and float(r.v_o.abs().max()) == 0
    b = _scene(8, 30, C=3, origin=spec.origin, dims=spec.dims, resolution=spec.resolution, smax=1.0)
    r = P.Voxelizer(spec, P.VoxelizeConfig(tau=float("inf")), 3)(b)
    assert bool((r.labels == r.free_code).all())
    classes = P.ClassTable(("a", "b", "c"), free_index=-1)
    prims = [P.SuperQuadric(mu=[0, 0, 0], scale=[1, 1, 1], rot=[1, 0, 0, 0], opacity=1.0,
                            logits=[0.0, 2.0, 1.0], eps1=1.0, eps2=1.0)]
    sem, dense = P.voxelize(P.Scene(prims, classes), spec)
    lab = np.asarray(sem.labels)
    assert lab.min() == -1 and set(np.unique(lab)) <= {-1, 1}
    assert lab[4, 4, 2] == 1


@pytest.mark.parametrize("n_prims", [256, 2000])
@pytest.mark.parametrize("stream", ["0", "1"])
def test_persistent_and_per_tile_evaluators_bit_identical(monkeypatch, n_prims, stream):
    """The persistent evaluator (work counter) and one CTA per work item run
    the same per-tile code: identical bits, for the chunk-staged kernel
    (SQV_STREAM=0, the default for sparse batches) and the streaming one
    (SQV_STREAM=1, the default for dense batches)."""
    P = _pkg()
    from paper_2511_17361_b200.scenegen import gen_frames
    spec = P.VoxelGridSpec()
    monkeypatch.setenv("SQV_STREAM", stream)
    for prec in ("strict", "fast"):
        cfg = P.VoxelizeConfig(precision=prec)
        b = gen_frames(31, 3, n_prims)
        outs = []
        for mode in ("1", "0"):
            monkeypatch.setenv("SQV_PERSIST", mode)
            r = P.Voxelizer(spec, cfg, 18)(b, dense=True)
            outs.append({k: getattr(r, k).cpu().numpy() for k in ("labels", "v_o", "v_c")})
        for k in ("labels", "v_o", "v_c"):
            np.testing.assert_array_equal(outs[0][k], outs[1][k], err_msg=f"{prec} {k}")


@pytest.mark.parametrize("case", range(int(os.environ.get("SQV_RANDOM_CASES", "40"))))
def test_randomized_configurations(case):
    """Sampled grid shapes (tile-ragged dims, offset origins, fine/coarse
    resolutions), class counts 1..24, both semantic modes, both precisions,
    truncated or not, ragged n_valid, persistent or per-tile evaluator:
    bins exact, densities and labels at the mode's tolerance."""
    P = _pkg()
    import os
    from paper_2511_17361_b200.core import PrimitiveBatch
    rng = np.random.default_rng(1000 + case)
    dims = (int(rng.integers(5, 45)), int(rng.integers(5, 45)), int(rng.integers(3, 36)))
    res = float(rng.choice([0.2, 0.37, 0.5]))
    origin = tuple(float(x) for x in rng.uniform(-6, 2, 3))
    C = int(rng.choice([1, 2, 5, 12, 17, 18, 19, 23, 24]))
    mode = "prob-sum" if rng.random() < 0.4 else "logit-sum"
    prec = "fast" if rng.random() < 0.3 else "strict"
    truncate = rng.random() < 0.75
    F, N = int(rng.integers(1, 4)), int(rng.integers(1, 60))
    hi = tuple(o + d * res for o, d in zip(origin, dims))
    spec = P.VoxelGridSpec(origin, dims, res)
    cfg = P.VoxelizeConfig(tau=float(rng.choice([0.0, 0.01, 0.2])),
                           neighborhood_radius=int(rng.integers(0, 6)), semantic_mode=mode,
                           precision=prec)
    b = _scene(77 + case, N, C, frames=F, origin=origin, dims=dims, resolution=res,
               smax=float(rng.choice([1.0, 4.0])))
    nv = rng.integers(0, N + 1, F).astype(np.int32)
    b = PrimitiveBatch(b.mu, b.scale, b.rot, b.opacity, b.eps, b.logits, n_valid=nv)
    # all four evaluator variants: persistent or per work item, chunk-staged
    # or streaming
    os.environ["SQV_PERSIST"] = str(case % 2)
    os.environ["SQV_STREAM"] = str((case // 2) % 2)
    os.environ["SQV_BIN"] = ("radix", "frame")[(case // 4) % 2]  # both binning paths
    try:
        out = _run(b, spec, cfg, C, truncate=truncate, bins=True)
    finally:
        del os.environ["SQV_PERSIST"]
        del os.environ["SQV_STREAM"]
        del os.environ["SQV_BIN"]
    ref, grid = _oracle(b, spec, cfg, out["free_code"], truncate=truncate)
    np.testing.assert_array_equal(out["windows"], ref["windows"])
    off, ids = O.bins(ref["windows"], grid.dims)
    np.testing.assert_array_equal(out["tile_off"], off)
    np.testing.assert_array_equal(out["prim_ids"], ids)
    assert out["n_pairs"] == ref["n_pairs"]
    # tiny grids: no agreement-rate floor (every mismatch must be explained)
    assert_parity(out, ref, cfg.tau, out["free_code"], mode=prec, min_agreement=0.0)


def test_run_many_two_stream_pipeline_matches_direct_calls():
    """Voxelizer.run_many (alternating streams, two workspaces and output
    slots) gives the same bits as one call per batch."""
    P = _pkg()
    import torch
    from paper_2511_17361_b200.scenegen import gen_frames
    spec, cfg = P.VoxelGridSpec(), P.VoxelizeConfig()
    vox = P.Voxelizer(spec, cfg, 18)
    batches = [vox.to_device(gen_frames(50 + k, 2, 300 + 200 * k)) for k in range(4)]
    direct = [vox(b, dense=True) for b in batches]
    want = [(r.labels.cpu().numpy(), r.v_c.cpu().numpy()) for r in direct]
    outs = [vox.alloc(2), vox.alloc(2)]
    got = []
    vox.run_many(batches, outs, on_device=lambda k, r: got.append(
        (r.labels.clone(), r.v_c.clone())))
    torch.cuda.synchronize()
    assert len(got) == 4
    for (gl, gc), (wl, wc) in zip(got, want):
        np.testing.assert_array_equal(gl.cpu().numpy(), wl)
        np.testing.assert_array_equal(gc.cpu().numpy(), wc)


@pytest.mark.parametrize("case", range(int(os.environ.get("SQV_RANDOM_DENSE_CASES", "8"))))
def test_randomized_dense_configurations(case):
    """Dense random scenes (hundreds of entries per tile: multi-chunk tiles,
    many K steps, all three strict-mode passes) vs the oracle."""
    P = _pkg()
    rng = np.random.default_rng(5000 + case)
    dims = (int(rng.integers(24, 72)), int(rng.integers(24, 72)), int(rng.choice([8, 16, 20])))
    res = float(rng.choice([0.3, 0.4]))
    origin = (-dims[0] * res / 2, -dims[1] * res / 2, -1.0)
    C = int(rng.choice([5, 12, 18, 24]))
    prec = "fast" if case % 3 == 2 else "strict"
    mode = "prob-sum" if case % 4 == 3 else "logit-sum"
    N = int(rng.integers(300, 1500))
    spec = P.VoxelGridSpec(origin, dims, res)
    cfg = P.VoxelizeConfig(semantic_mode=mode, precision=prec)
    b = _scene(9000 + case, N, C, frames=2, origin=origin, dims=dims, resolution=res,
               emin=float(rng.choice([0.1, 0.2])))
    os.environ["SQV_PERSIST"] = str(case % 2)  # deep tiles in every evaluator variant
    os.environ["SQV_STREAM"] = str((case // 2) % 2)
    os.environ["SQV_BIN"] = ("radix", "frame", "fused")[(case // 4) % 3]
    try:
        out = _run(b, spec, cfg, C, bins=True)
    finally:
        del os.environ["SQV_PERSIST"]
        del os.environ["SQV_STREAM"]
        del os.environ["SQV_BIN"]
    ref, grid = _oracle(b, spec, cfg, out["free_code"])
    off, ids = O.bins(ref["windows"], grid.dims)
    np.testing.assert_array_equal(out["tile_off"], off)
    np.testing.assert_array_equal(out["prim_ids"], ids)
    assert out["n_pairs"] == ref["n_pairs"]
    assert_parity(out, ref, cfg.tau, out["free_code"], mode=prec)


@pytest.mark.parametrize("scale", [1.0, 1e6, 1e9])
def test_block_cull_bound_with_large_logits(scale):
    """The block cull drops weights below exp(-cut) with a per-primitive cut
    = max(36, ln(N wmax / 2e-12)) (sqv_common.cuh kBlockCutMin): with small
    primitives (most window voxels deep in the tail, F in 36..87), tau = 0
    (every voxel labelled, tail voxels included) and logits scaled up to
    1e9, v_o, v_c and labels still meet the parity bound."""
    P = _pkg()
    from paper_2511_17361_b200.core import PrimitiveBatch
    origin, dims, res = (-8.0, -8.0, -1.0), (40, 40, 16), 0.4
    spec = P.VoxelGridSpec(origin, dims, res)
    cfg = P.VoxelizeConfig(tau=0.0, neighborhood_radius=5, semantic_mode="logit-sum")
    b = _scene(4242, 60, 18, origin=origin, dims=dims, resolution=res, smax=0.6)
    b = PrimitiveBatch(b.mu, b.scale, b.rot, b.opacity, b.eps, b.logits * scale)
    out = _run(b, spec, cfg, 18)
    ref, _ = _oracle(b, spec, cfg, out["free_code"])
    assert out["n_pairs"] == ref["n_pairs"]
    # tau = 0 labels every voxel; voxels whose whole oracle v_o is below the
    # cull's drop bound may lose every contribution (v_c = 0 -> label 0):
    # allowed by the near-tie rule (gap < 2 * 2e-12), and excluded from the
    # agreement rate, which must still reach 99.99% on the rest
    _, lab = assert_parity(out, ref, cfg.tau, out["free_code"])
    assert lab["n_resolvable"] > 0.5 * out["labels"].size


def test_entry_total_past_2_31_reports_split_frames():
    """The bin entry total is summed in 64 bits by prep: a batch
    past 2^31 entries fails with the 'split frames' error before the int32
    scan offsets reach emit — not a wrapped total (a bogus workspace size,
    or out-of-bounds emit stores).  5,000 untruncated primitives on a
    4096x4096x16 grid (262,144 tiles per frame) x 2 frames = 2.6e9 entries;
    only prep and the scan run, so the call is cheap."""
    import ctypes
    import torch
    P = _pkg()
    from paper_2511_17361_b200 import _lib
    from paper_2511_17361_b200.scenegen import gen_frames_device
    spec = P.VoxelGridSpec((-40.0, -40.0, -1.0), (4096, 4096, 16), 0.4)
    b = gen_frames_device(3, 2, 5000, 4, origin=spec.origin, dims=spec.dims,
                          resolution=spec.resolution)
    L = _lib.lib()
    Pr = _lib.Prims()
    Pr.mu, Pr.scale, Pr.rot = b.mu.data_ptr(), b.scale.data_ptr(), b.rot.data_ptr()
    Pr.opacity, Pr.eps, Pr.logits = b.opacity.data_ptr(), b.eps.data_ptr(), b.logits.data_ptr()
    Pr.n_valid = None
    Pr.n_frames, Pr.n_prims, Pr.n_classes = 2, 5000, 4
    cfg = _lib.Cfg()
    cfg.tau, cfg.neighborhood_radius, cfg.truncate = 0.01, 5, 0
    cfg.semantic_mode, cfg.free_label, cfg.window_extent, cfg.precision = 0, 255, 2.5, 1
    grid = spec._c()
    dummy = torch.empty(16, dtype=torch.uint8, device="cuda")
    O_ = _lib.Outputs()
    O_.labels = dummy.data_ptr()
    fixed = int(L.sqv_workspace_bytes(2, 5000, 4, ctypes.byref(grid), 0))
    ws = torch.empty(fixed, dtype=torch.uint8, device="cuda")
    need = ctypes.c_size_t(0)
    bp, bb = ctypes.c_int64(0), ctypes.c_int32(0)
    rc = L.sqv_voxelize(ctypes.byref(Pr), ctypes.byref(grid), ctypes.byref(cfg),
                        ctypes.byref(O_), None, ws.data_ptr(), ws.numel(), ctypes.byref(need),
                        ctypes.byref(bp), ctypes.byref(bb), _lib.stream_ptr())
    torch.cuda.synchronize()
    msg = _lib.last_error()
    assert rc == _lib.SQV_ERR_ARG, (rc, msg)
    assert "split frames" in msg, msg
    E = int(re.search(r"entries: (\d+)", msg).group(1))
    tiles = 512 * 512
    assert E == 2 * 5000 * tiles  # untruncated: every primitive overlaps every tile


def test_torch_ops_match_the_package_api():
    """torch.ops.sqocc.voxelize / prep_bin / confusion give the bits of
    Voxelizer and confusion_matrix, and pass torch.library.opcheck's schema
    and fake-tensor checks."""
    import torch
    P = _pkg()
    from paper_2511_17361_b200 import torch_ops  # noqa: F401
    from paper_2511_17361_b200.metrics import confusion_matrix
    from paper_2511_17361_b200.scenegen import gen_frames
    spec = P.VoxelGridSpec((-10.0, -9.0, -1.0), (52, 44, 20), 0.4)
    b = gen_frames(77, 2, 300, 12, origin=spec.origin, dims=spec.dims, resolution=spec.resolution)
    vox = P.Voxelizer(spec, P.VoxelizeConfig(), 12)
    db = vox.to_device(b)
    args = (db.mu, db.scale, db.rot, db.opacity, db.eps, db.logits, list(spec.origin),
            list(spec.dims), spec.resolution)
    lab, vo, vc = torch.ops.sqocc.voxelize(*args)
    r = vox(db, dense=True, bins=True)
    for x, y in ((lab, r.labels), (vo, r.v_o), (vc, r.v_c)):
        assert torch.equal(x, y)
    w, to, ids, n = torch.ops.sqocc.prep_bin(*args)
    assert torch.equal(w, r.bins["windows"]) and torch.equal(to, r.bins["tile_off"])
    assert torch.equal(ids, r.bins["prim_ids"]) and int(n) == r.n_pairs
    gt = torch.roll(lab, 1, dims=-1).contiguous()
    assert torch.equal(torch.ops.sqocc.confusion(lab, gt, 12), confusion_matrix(lab, gt, 12))
    utils = ("test_schema", "test_faketensor")
    torch.library.opcheck(torch.ops.sqocc.voxelize.default, args, test_utils=utils)
    torch.library.opcheck(torch.ops.sqocc.confusion.default, (lab, gt, 12), test_utils=utils)


def test_evaluator_work_counters():
    """sqv_stats_attach: MUFU ops and evaluated pairs of the evaluators, whole
    128-voxel warp blocks, between 4 and 7 MUFU per evaluated pair (strict),
    fewer evaluated pairs than the window pairs they were culled from."""
    import torch
    P = _pkg()
    from paper_2511_17361_b200 import _lib
    from paper_2511_17361_b200.scenegen import gen_frames
    vox = P.Voxelizer(P.VoxelGridSpec(), P.VoxelizeConfig(), 18)
    b = vox.to_device(gen_frames(4, 2, 2000, 18))
    st = torch.zeros(2, dtype=torch.int64, device="cuda")
    _lib.stats_attach(st)
    try:
        r = vox(b, dense=False)
        torch.cuda.synchronize()
    finally:
        _lib.stats_attach(None)
    mufu, pairs = (int(v) for v in st.cpu().tolist())
    assert pairs > 0 and pairs % 128 == 0
    assert 4 * pairs <= mufu <= 7 * pairs
    assert 0.5 * r.n_pairs < pairs < r.n_pairs
    vox(b, dense=False)  # detached: counters unchanged
    torch.cuda.synchronize()
    assert int(st[0]) == mufu


@pytest.mark.parametrize("n_prims", [256, 2000])
def test_binning_paths_bit_identical(monkeypatch, n_prims):
    """Per-frame counting-sort binning (sqv_bin.cu, with and without the
    fused block masks) and emit + radix sort give the same bins, masks and
    outputs bit for bit."""
    P = _pkg()
    from paper_2511_17361_b200.scenegen import gen_frames
    spec = P.VoxelGridSpec()
    b = gen_frames(71, 3, n_prims)
    outs = []
    for mode in ("radix", "frame", "fused"):
        monkeypatch.setenv("SQV_BIN", mode)
        r = P.Voxelizer(spec, P.VoxelizeConfig(), 18)(b, dense=True, bins=True)
        outs.append([r.labels.cpu().numpy(), r.v_c.cpu().numpy(),
                     *(r.bins[k].cpu().numpy() for k in ("windows", "tile_off", "prim_ids"))])
    for o in outs[1:]:
        for x, y in zip(outs[0], o):
            np.testing.assert_array_equal(x, y)
