"""Generate the golden fixtures that pin the CPU oracle to the reference.

Run HERE (needs /root/reference, read-only):  python tests/golden/make_golden.py

The reference ships the per-point math (sqocc.core) but no voxelizer, so:

* ``core_pairs.npz``   — the reference's own ``SuperQuadric`` construction
  (validation, quaternion normalisation, eps clamp; core.py:143-173),
  ``to_local`` (core.py:237-244), ``inside_outside`` (core.py:254-273) and
  ``density`` (core.py:276-282) evaluated on seeded primitives and points.
* ``voxelize_*.npz``   — small scenes voxelized with the reference's
  ``density()`` per primitive, glued by the SPEC rules written out below
  (window SPEC.md:348 + ledger :382, sample point :384, sigma=0 skip :349,
  scatter v_o/v_c :348, prob-sum :383, finalize :365-369, bins :385 with the
  tile shape of include/sqv.h).
* ``confusion.npz``    — seeded label-grid pairs with confusion counts computed
  by direct enumeration ("confusion-matrix oracle").

All inputs are stored raw (before clamping / normalisation) so every consumer
re-runs the full path.  The fixtures are small; regenerate only when the
generator changes.
"""
from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
TILE = (8, 8, 16)


def _ref():
    sys.path.insert(0, REF_SRC)
    from sqocc import core  # noqa: E402  (the reference, imported read-only)
    return core


def raw_prims(rng, n, C, lo, hi, smin=0.2, smax=2.0, emin=0.1, emax=2.5):
    mu = rng.uniform(lo, hi, size=(n, 3))
    scale = rng.uniform(smin, smax, size=(n, 3))
    rot = rng.normal(size=(n, 4)) * rng.uniform(0.5, 2.0, size=(n, 1))  # unnormalised on purpose
    opacity = rng.uniform(0.0, 1.0, size=n)
    eps = rng.uniform(emin, emax, size=(n, 2))
    logits = rng.normal(size=(n, C))
    return mu, scale, rot, opacity, eps, logits


def build_sqs(core, mu, scale, rot, opacity, eps, logits):
    return [core.SuperQuadric(mu=mu[i], scale=scale[i], rot=rot[i], opacity=opacity[i],
                              logits=logits[i], eps1=eps[i, 0], eps2=eps[i, 1])
            for i in range(len(opacity))]


def gen_core_pairs(core):
    rng = np.random.default_rng(20251117)
    n, C, per = 256, 4, 24
    mu, scale, rot, opacity, eps, logits = raw_prims(rng, n, C, -5.0, 5.0, 0.05, 4.0, 0.05, 3.0)
    sqs = build_sqs(core, mu, scale, rot, opacity, eps, logits)
    prim = np.repeat(np.arange(n), per).astype(np.int32)
    pts = np.empty((n * per, 3))
    loc = np.empty((n * per, 3))
    F = np.empty(n * per)
    dens = np.empty(n * per)
    for i, sq in enumerate(sqs):
        # points at 0.1 .. 3 semi-axes in random local directions, plus the centre
        d = rng.normal(size=(per, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        r = rng.uniform(0.1, 3.0, size=(per, 1)) * sq.scale[None, :]
        xl = d * r
        xl[0] = 0.0
        xw = core.to_world(sq, xl)
        sl = slice(i * per, (i + 1) * per)
        pts[sl] = xw
        loc[sl] = core.to_local(sq, xw)
        F[sl] = core.inside_outside(sq, loc[sl])
        dens[sl] = core.density(sq, xw)
    clamped = np.array([sq.eps_clamped for sq in sqs])
    eps_after = np.array([[sq.eps1, sq.eps2] for sq in sqs])
    rot_after = np.array([sq.rot for sq in sqs])
    np.savez_compressed(os.path.join(OUT, "core_pairs.npz"), mu=mu, scale=scale, rot=rot,
                        opacity=opacity, eps=eps, logits=logits, pair_prim=prim, points=pts,
                        local=loc, F=F, density=dens, eps_clamped=clamped,
                        eps_after=eps_after, rot_after=rot_after)
    return len(F)


def ref_voxelize(core, sqs, origin, dims, res, tau, radius, truncate, prob_sum, free_label,
                 extent=2.5):
    """SPEC.md:345-369 glue over the reference's density()."""
    origin = np.asarray(origin, np.float64)
    dims = np.asarray(dims, np.int64)
    nx, ny, nz = (int(d) for d in dims)
    C = sqs[0].num_classes if sqs else 1
    v_o = np.zeros((nz, ny, nx))
    v_c = np.zeros((nz, ny, nx, C))
    windows = np.zeros((len(sqs), 6), np.int32)
    windows[:, :3] = 1
    pairs = 0
    for i, sq in enumerate(sqs):
        if truncate:
            c = np.floor((sq.mu - origin) / res)
            r = radius + np.ceil(sq.scale.max() * extent / res)
            lo = np.maximum(c - r, 0.0)
            hi = np.minimum(c + r, (dims - 1).astype(np.float64))
        else:
            lo = np.zeros(3)
            hi = (dims - 1).astype(np.float64)
        if sq.opacity == 0.0 or np.any(lo > hi):      # SPEC.md:349 sigma=0 skipped
            continue
        lo = lo.astype(np.int64)
        hi = hi.astype(np.int64)
        windows[i, :3], windows[i, 3:] = lo, hi
        zz, yy, xx = np.meshgrid(np.arange(lo[2], hi[2] + 1), np.arange(lo[1], hi[1] + 1),
                                 np.arange(lo[0], hi[0] + 1), indexing="ij")
        idx = np.stack([xx.ravel(), yy.ravel(), zz.ravel()], axis=1)
        p = origin + (idx + 0.5) * res                  # voxel centres
        w = core.density(sq, p)                          # the reference's Eq. 4
        if prob_sum:
            e = np.exp(sq.logits - sq.logits.max())
            cw = e / e.sum()
        else:
            cw = sq.logits
        # per-voxel accumulation in primitive order (np.add.at keeps it unbuffered)
        np.add.at(v_o, (idx[:, 2], idx[:, 1], idx[:, 0]), sq.opacity * w)
        np.add.at(v_c, (idx[:, 2], idx[:, 1], idx[:, 0]), w[:, None] * cw[None, :])
        pairs += len(w)
    labels = np.where(v_o < tau, free_label, np.argmax(v_c, axis=-1)).astype(np.uint8)
    return v_o.reshape(-1), v_c.reshape(-1, C), labels.reshape(-1), windows, pairs


def ref_bins(windows, dims):
    ntx, nty, ntz = ((d + t - 1) // t for d, t in zip(dims, TILE))
    lists = [[] for _ in range(ntx * nty * ntz)]
    for i, w in enumerate(windows):
        if w[0] > w[3] or w[1] > w[4] or w[2] > w[5]:
            continue
        for tz in range(w[2] // TILE[2], w[5] // TILE[2] + 1):
            for ty in range(w[1] // TILE[1], w[4] // TILE[1] + 1):
                for tx in range(w[0] // TILE[0], w[3] // TILE[0] + 1):
                    lists[tx + ntx * (ty + nty * tz)].append(i)
    off = np.zeros(len(lists) + 1, np.int32)
    off[1:] = np.cumsum([len(l) for l in lists])
    ids = np.array([i for l in lists for i in l], np.int32)
    return off, ids


SCENES = [
    # name, seed, n, C, origin, dims, res, tau, radius, truncate, prob_sum, free, gen kwargs
    ("basic", 1, 12, 5, (-4.0, -4.0, -3.0), (24, 20, 18), 0.35, 0.01, 5, True, False, 5, {}),
    ("bruteforce", 2, 10, 5, (-4.0, -4.0, -3.0), (24, 20, 18), 0.35, 0.01, 5, False, False, 5, {}),
    ("probsum", 3, 14, 3, (-3.0, -5.0, -2.0), (20, 26, 12), 0.4, 0.02, 3, True, True, 3, {}),
    ("ragged_edges", 4, 30, 4, (-6.0, -6.0, -2.0), (21, 13, 7), 0.5, 0.01, 2, True, False, 200,
     dict(margin=3.0, zero_sigma=4)),
    ("stress_eps", 5, 20, 6, (-4.0, -4.0, -2.0), (16, 16, 16), 0.3, 0.005, 5, True, False, 6,
     dict(emin=0.05, emax=3.0, smin=0.05, smax=1.5)),
    ("tau0", 6, 6, 2, (-3.0, -3.0, -3.0), (12, 12, 12), 0.5, 0.0, 1, True, False, 2, {}),
]


def gen_voxelize(core):
    names = []
    for (name, seed, n, C, origin, dims, res, tau, radius, truncate, prob_sum, free,
         kw) in SCENES:
        rng = np.random.default_rng(1000 + seed)
        lo = np.asarray(origin)
        hi = lo + np.asarray(dims) * res
        margin = kw.get("margin", 0.0)
        mu, scale, rot, opacity, eps, logits = raw_prims(
            rng, n, C, lo - margin, hi + margin, kw.get("smin", 0.2), kw.get("smax", 2.0),
            kw.get("emin", 0.1), kw.get("emax", 2.5))
        zs = kw.get("zero_sigma", 0)
        if zs:
            opacity[rng.choice(n, zs, replace=False)] = 0.0
        sqs = build_sqs(core, mu, scale, rot, opacity, eps, logits)
        v_o, v_c, labels, windows, pairs = ref_voxelize(core, sqs, origin, dims, res, tau,
                                                        radius, truncate, prob_sum, free)
        off, ids = ref_bins(windows, dims)
        np.savez_compressed(os.path.join(OUT, f"voxelize_{name}.npz"), mu=mu, scale=scale,
                            rot=rot, opacity=opacity, eps=eps, logits=logits,
                            origin=np.asarray(origin, np.float64),
                            dims=np.asarray(dims, np.int32), res=res, tau=tau, radius=radius,
                            truncate=truncate, prob_sum=prob_sum, free_label=free, v_o=v_o,
                            v_c=v_c, labels=labels, windows=windows, tile_off=off, prim_ids=ids,
                            n_pairs=pairs)
        names.append((name, pairs))
    return names


def gen_confusion():
    rng = np.random.default_rng(77)
    preds, gts, cms, Cs = [], [], [], []
    for k in range(50):                      # 50 seeded grid pairs
        C = int(rng.integers(1, 19))
        free = 255
        n = int(rng.integers(1, 600))
        pool = np.concatenate([np.arange(C), [free]]).astype(np.uint8)
        gt = rng.choice(pool, size=n)
        pred = np.where(rng.uniform(size=n) < 0.6, gt, rng.choice(pool, size=n)).astype(np.uint8)
        cm = np.zeros((C + 1, C + 1), np.int64)
        for g, p in zip(gt, pred):           # direct enumeration
            cm[min(int(g), C), min(int(p), C)] += 1
        preds.append(pred)
        gts.append(gt)
        cms.append(cm.ravel())
        Cs.append(C)
    lens = np.array([len(p) for p in preds])
    np.savez_compressed(os.path.join(OUT, "confusion.npz"), pred=np.concatenate(preds),
                        gt=np.concatenate(gts), lens=lens, C=np.array(Cs),
                        cm=np.concatenate(cms))


def main():
    core = _ref()
    print("core pairs:", gen_core_pairs(core))
    for name, pairs in gen_voxelize(core):
        print(f"voxelize_{name}: {pairs} pairs")
    gen_confusion()
    print("confusion: 50 pairs")


if __name__ == "__main__":
    main()
