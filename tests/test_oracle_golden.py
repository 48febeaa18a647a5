"""Pin the CPU oracle (oracle/sqv_oracle.c) to the reference's own outputs.

Fixtures come from tests/golden/make_golden.py, which runs the reference's
sqocc.core (/root/reference/pkg/src/sqocc/core.py) on seeded inputs.
"""
import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden
from oracle import oracle as O


def _prims(g, F1=True):
    return O.Prims.of(type("B", (), {k: g[k] for k in
                                     ("mu", "scale", "rot", "opacity", "eps", "logits")}))


def test_core_pairs_F_and_density_match_reference():
    g = load_golden("core_pairs.npz")
    p = _prims(g)
    F, d = O.density(p, g["points"], g["pair_prim"])
    np.testing.assert_allclose(F, g["F"], rtol=1e-12, atol=1e-300)
    # exp(-F) amplifies F's last-bit differences by F: relative 1e-12 per unit of F
    rel = np.abs(d - g["density"]) / np.maximum(g["density"], 1e-300)
    assert np.all(rel <= 1e-12 * np.maximum(1.0, g["F"]))


def test_spec_known_answers():
    # SPEC.md:75-78 (inside_outside), :86-88 (density), :65-66 (to_local)
    def one(mu, scale, rot, e1, e2, pts):
        p = O.Prims.of(type("B", (), dict(mu=np.array([mu], float), scale=np.array([scale], float),
                                          rot=np.array([rot], float), opacity=np.array([1.0]),
                                          eps=np.array([[e1, e2]]), logits=np.zeros((1, 1)))))
        return O.density(p, np.array(pts, float), np.zeros(len(pts), np.int32))
    F, d = one([0, 0, 0], [1, 1, 1], [1, 0, 0, 0], 1, 1, [[1, 0, 0], [0, 0, 0], [2, 0, 0]])
    np.testing.assert_allclose(F, [1.0, 0.0, 4.0], rtol=1e-15)
    np.testing.assert_allclose(d, [np.exp(-1.0), 1.0, np.exp(-4.0)], rtol=1e-15)
    F, _ = one([0, 0, 0], [1.0, 0.7, 0.5], [1, 0, 0, 0], 0.6, 0.7, [[1, 0, 0]])  # Fig. 3 shape
    np.testing.assert_allclose(F, [1.0], rtol=1e-15)
    # 90 deg about z (local-to-world): world (0,1,0) is local (1,0,0) -> F = 1 for unit sphere
    c = np.cos(np.pi / 4)
    F, _ = one([0, 0, 0], [1, 2, 3], [c, 0, 0, c], 1, 1, [[0, 1, 0]])
    np.testing.assert_allclose(F, [1.0], rtol=1e-12)


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "voxelize_*.npz"))),
                         ids=lambda p: os.path.basename(p)[9:-4])
def test_voxelize_matches_reference_glue(path):
    g = dict(np.load(path))
    p = _prims(g)
    grid = O.Grid(tuple(g["origin"]), tuple(int(x) for x in g["dims"]), float(g["res"]))
    cfg = O.Cfg(float(g["tau"]), int(g["radius"]), bool(g["truncate"]), bool(g["prob_sum"]),
                int(g["free_label"]))
    win = O.prep(p, grid, cfg)[0]
    np.testing.assert_array_equal(win, g["windows"])
    off, ids = O.bins(win[None], grid.dims)
    np.testing.assert_array_equal(off, g["tile_off"])
    np.testing.assert_array_equal(ids, g["prim_ids"])
    r = O.voxelize(p, grid, cfg)
    assert r["n_pairs"] == int(g["n_pairs"])
    np.testing.assert_allclose(r["v_o"][0], g["v_o"], rtol=1e-12, atol=1e-300)
    np.testing.assert_allclose(r["v_c"][0], g["v_c"], rtol=1e-11, atol=1e-13)
    np.testing.assert_array_equal(r["labels"][0], g["labels"])


def test_confusion_matches_enumeration():
    g = load_golden("confusion.npz")
    s = 0
    c0 = 0
    for n, C in zip(g["lens"], g["C"]):
        k = (C + 1) ** 2
        cm = O.confusion(g["pred"][s:s + n], g["gt"][s:s + n], int(C))
        np.testing.assert_array_equal(cm.ravel(), g["cm"][c0:c0 + k])
        s += n
        c0 += k


def test_oracle_thread_count_determinism():
    g = load_golden("voxelize_basic.npz")
    p = _prims(g)
    grid = O.Grid(tuple(g["origin"]), tuple(int(x) for x in g["dims"]), float(g["res"]))
    cfg = O.Cfg(float(g["tau"]), int(g["radius"]), True, False, int(g["free_label"]))
    n0 = O.threads()
    try:
        O.set_threads(1)
        a = O.voxelize(p, grid, cfg)
        O.set_threads(max(2, n0))
        b = O.voxelize(p, grid, cfg)
    finally:
        O.set_threads(n0)
    assert np.array_equal(a["v_o"], b["v_o"]) and np.array_equal(a["v_c"], b["v_c"])
