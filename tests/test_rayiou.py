"""ray_iou: the oracle on the SPEC examples and properties
(CPU), the device kernel against the oracle bit-for-bit (GPU)."""
import numpy as np
import pytest

import paper_2511_17361_b200 as P
from oracle import oracle as O
from paper_2511_17361_b200 import metrics as M

THR = (1.0, 2.0, 4.0)


def _axis_case():
    """single-axis ray, pred hit at 10.0 m, gt at 11.5 m, same class."""
    dims, org, res = (40, 4, 4), (0.0, 0.0, 0.0), 0.5
    pred = np.full((4, 4, 40), 255, np.uint8)
    gt = pred.copy()
    pred[2, 2, 20] = 3
    gt[2, 2, 23] = 3
    return dims, org, res, pred.ravel(), gt.ravel(), [[0.0, 1.25, 1.25]], [[1.0, 0.0, 0.0]]


def _random_case(seed, F=3, dims=(37, 29, 11), C=5, fill=0.04):
    rng = np.random.default_rng(seed)
    V = int(np.prod(dims))
    lab = lambda: np.where(rng.random((F, V)) < fill, rng.integers(0, C, (F, V)), 255).astype(
        np.uint8)
    pred, gt = lab(), lab()
    gt = np.where(rng.random((F, V)) < 0.7, pred, gt).astype(np.uint8)  # correlated grids
    org, res = (-3.3, 1.7, -0.9), 0.37
    spec = P.VoxelGridSpec(origin=org, dims=dims, resolution=res)
    o1, d1 = M.default_rays(spec, n_azimuth=90, elevations_deg=(-20.0, -3.0, 0.0, 7.0))
    n = 300
    o2 = np.array(org) + rng.uniform(-2, 1.2, (n, 3)) * np.array(dims) * res
    d2 = rng.normal(size=(n, 3))
    d2[:40, 1:] = 0.0          # axis-aligned
    d2[40:80, 2] = 0.0         # in a z plane
    d2 /= np.linalg.norm(d2, axis=1, keepdims=True)
    # origins exactly on voxel faces
    o3 = np.array(org) + rng.integers(0, 10, (40, 3)) * res
    d3 = rng.normal(size=(40, 3))
    d3 /= np.linalg.norm(d3, axis=1, keepdims=True)
    return (spec, C, pred, gt, np.concatenate([o1, o2, o3]), np.concatenate([d1, d2, d3]))


def test_oracle_spec_examples():
    dims, org, res, pred, gt, o, d = _axis_case()
    c, h = O.ray_iou(pred, gt, dims, org, res, 5, o, d, THR)
    assert h["d_pred"][0, 0] == 10.0 and h["d_gt"][0, 0] == 11.5
    np.testing.assert_array_equal(c, [[0, 1, 1], [1, 0, 0], [1, 0, 0]])
    r = M.rayiou_from_counts(c, THR)
    assert r == {1.0: 0.0, 2.0: 1.0, 4.0: 1.0}
    # pred = gt -> 1.0 at all thresholds; pred empty, gt hit -> 0.0
    c, _ = O.ray_iou(gt, gt, dims, org, res, 5, o, d, THR)
    assert M.rayiou_from_counts(c, THR) == {1.0: 1.0, 2.0: 1.0, 4.0: 1.0}
    empty = np.full_like(gt, 255)
    c, _ = O.ray_iou(empty, gt, dims, org, res, 5, o, d, THR)
    assert M.rayiou_from_counts(c, THR) == {1.0: 0.0, 2.0: 0.0, 4.0: 0.0}


def test_oracle_monotone_in_threshold_and_self_iou():
    spec, C, pred, gt, o, d = _random_case(1)
    c, h = O.ray_iou(pred, gt, spec.dims, spec.origin, spec.resolution, C, o, d, THR)
    r = M.rayiou_from_counts(c, THR)
    assert r[1.0] <= r[2.0] <= r[4.0]
    assert (h["c_pred"] >= 0).mean() > 0.3  # the case exercises hits
    c, _ = O.ray_iou(pred, pred, spec.dims, spec.origin, spec.resolution, C, o, d, THR)
    assert (c[:, 1:] == 0).all()


def test_default_rays_and_validation():
    o, d = M.default_rays(P.VoxelGridSpec())
    assert o.shape == d.shape == (1440, 3)
    np.testing.assert_allclose(np.linalg.norm(d, axis=1), 1.0)
    np.testing.assert_allclose(o[0], [0.0, 0.0, 2.2])
    with pytest.raises(ValueError, match="zero rays"):
        M.ray_counts(np.zeros(640000, np.uint8), np.zeros(640000, np.uint8), P.VoxelGridSpec(),
                     18, np.zeros((0, 3)), np.zeros((0, 3)))
    with pytest.raises(ValueError, match="unit"):
        M.ray_counts(np.zeros(640000, np.uint8), np.zeros(640000, np.uint8), P.VoxelGridSpec(),
                     18, [[0, 0, 0]], [[2.0, 0, 0]])


@pytest.mark.gpu
def test_gpu_ray_iou_matches_oracle_bitwise():
    spec, C, pred, gt, o, d = _random_case(7)
    want_c, want_h = O.ray_iou(pred, gt, spec.dims, spec.origin, spec.resolution, C, o, d, THR)
    got_c, got_h = M.ray_counts(pred, gt, spec, C, o, d, THR, return_hits=True)
    for k in ("d_pred", "c_pred", "d_gt", "c_gt"):
        np.testing.assert_array_equal(got_h[k].cpu().numpy(), want_h[k], err_msg=k)
    np.testing.assert_array_equal(got_c.cpu().numpy(), want_c)


@pytest.mark.gpu
def test_gpu_ray_iou_spec_examples_and_grids():
    dims, org, res, pred, gt, o, d = _axis_case()
    spec = P.VoxelGridSpec(origin=org, dims=dims, resolution=res)
    c = M.ray_counts(pred, gt, spec, 5, o, d, THR).cpu().numpy()
    assert M.rayiou_from_counts(c, THR) == {1.0: 0.0, 2.0: 1.0, 4.0: 1.0}
    # SemanticGrid API on voxelized scenes: self = 1.0, monotone, = oracle
    from paper_2511_17361_b200.scenegen import gen_scene
    a = P.voxelize(gen_scene(3, 200), P.VoxelGridSpec(), P.VoxelizeConfig())[0]
    b = P.voxelize(gen_scene(4, 200), P.VoxelGridSpec(), P.VoxelizeConfig())[0]
    assert P.ray_iou(a, a) == {1.0: 1.0, 2.0: 1.0, 4.0: 1.0}
    r = P.ray_iou(a, b)
    assert r[1.0] <= r[2.0] <= r[4.0]
    flat = lambda g: np.where(np.asarray(g.labels) < 18, g.labels, 255).astype(
        np.uint8).transpose(2, 1, 0).ravel()
    oo, dd = M.default_rays(a.spec)
    c, _ = O.ray_iou(flat(a), flat(b), a.spec.dims, a.spec.origin, a.spec.resolution, 18, oo, dd,
                     THR)
    assert r == M.rayiou_from_counts(c, THR)
