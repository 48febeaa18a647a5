"""Device-side scene generation (sqv_gen_frames)."""
import numpy as np
import pytest

import paper_2511_17361_b200 as P
from philox_mirror import gen as mirror


def test_mirror_distributions():
    mu, scale, rot, op, eps, lg = mirror(7, 3, 4000, 18, (-40, -40, -1), (40, 40, 5.4), 0.2, 4.0,
                                         0.2)
    assert mu.shape == (3, 4000, 3) and lg.shape == (3, 4000, 18)
    assert (mu[..., 0] >= -40).all() and (mu[..., 2] < 5.4).all()
    assert (scale >= 0.2).all() and (scale < 4.0).all() and (eps >= 0.2).all()
    np.testing.assert_allclose(np.linalg.norm(rot, axis=-1), 1.0, rtol=1e-14)
    assert abs(lg.mean()) < 0.02 and abs(lg.std() - 1.0) < 0.02
    assert abs(op.mean() - 0.5) < 0.01
    # frame f of first_frame 0 == frame 0 of first_frame f
    a = mirror(7, 3, 50, 5, (0, 0, 0), (1, 1, 1), 0.2, 4.0, 0.2)
    b = mirror(7, 1, 50, 5, (0, 0, 0), (1, 1, 1), 0.2, 4.0, 0.2, first_frame=2)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x[2], y[0])


@pytest.mark.gpu
def test_device_generator_matches_mirror_and_voxelizes():
    from paper_2511_17361_b200.scenegen import gen_frames_device
    seed = (1 << 40) + 12345
    b = gen_frames_device(seed, 4, 3000, 18, first_frame=9)
    want = mirror(seed, 4, 3000, 18, (-40.0, -40.0, -1.0), (40.0, 40.0, 5.4), 0.2, 4.0, 0.2,
                  first_frame=9)
    got = [getattr(b, k).cpu().numpy() for k in ("mu", "scale", "rot", "opacity", "eps",
                                                 "logits")]
    for k in (0, 1, 3, 4):  # uniform-derived: bit-exact
        np.testing.assert_array_equal(got[k], want[k])
    np.testing.assert_allclose(got[2], want[2], rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(got[5], want[5], rtol=1e-12, atol=1e-14)
    # deterministic, and the batch goes straight into the voxelizer
    b2 = gen_frames_device(seed, 4, 3000, 18, first_frame=9)
    assert all((getattr(b, k) == getattr(b2, k)).all() for k in P.PrimitiveBatch.FIELDS)
    vox = P.Voxelizer(P.VoxelGridSpec(), P.VoxelizeConfig(), 18)
    r = vox(b, dense=False)
    assert r.n_pairs > 0 and r.labels.shape == (4, 16, 200, 200)


@pytest.mark.gpu
def test_evaluate_generated_independent_of_batching_and_shards():
    """The ground-truth jitter is keyed per frame, so the full confusion
    matrix is identical for any frames_per_batch, and shard matrices sum to
    the whole (what the NCCL all-reduce computes for any GPU count)."""
    from paper_2511_17361_b200 import distributed as D
    vox = P.Voxelizer(P.VoxelGridSpec(), P.VoxelizeConfig(), 18)
    whole = D.evaluate_generated(vox, 5, 6, 400, frames_per_batch=6).cpu().numpy()
    assert whole.sum() == 6 * 640000
    for fpb in (1, 2, 4):
        other = D.evaluate_generated(vox, 5, 6, 400, frames_per_batch=fpb).cpu().numpy()
        np.testing.assert_array_equal(whole, other, err_msg=f"frames_per_batch={fpb}")
    for world in (2, 4):
        parts = sum(D.evaluate_generated(vox, 5, 6, 400, frames_per_batch=3,
                                         frame_range=D.shard_frames(6, r, world)).cpu().numpy()
                    for r in range(world))
        np.testing.assert_array_equal(whole, parts, err_msg=f"world={world}")
    # the jitter is a real perturbation: gt differs from the prediction
    assert np.trace(whole) < whole.sum()


@pytest.mark.gpu
def test_gt_jitter_keyed_per_frame():
    from paper_2511_17361_b200.distributed import gt_jitter_device
    a_mu, a_lg = gt_jitter_device(11, 0, 5, 300, 18)
    b_mu, b_lg = gt_jitter_device(11, 3, 2, 300, 18)
    np.testing.assert_array_equal(a_mu[3:].cpu().numpy(), b_mu.cpu().numpy())
    np.testing.assert_array_equal(a_lg[3:].cpu().numpy(), b_lg.cpu().numpy())
    assert a_mu.shape == (5, 300, 3) and a_lg.shape == (5, 300, 18)
    assert abs(float(a_lg.std()) - 1.0) < 0.05
