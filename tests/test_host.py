"""CPU tests: host types, the C ABI surface, sharding/all-reduce (gloo), metrics folds."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT

import paper_2511_17361_b200 as P
from paper_2511_17361_b200 import _lib, metrics as M
from paper_2511_17361_b200.core import validation_bits
from paper_2511_17361_b200.distributed import shard_frames
from paper_2511_17361_b200.scenegen import gen_frames


def test_header_declares_exactly_the_exported_symbols():
    hdr = open(os.path.join(ROOT, "include", "sqv.h")).read()
    declared = set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(sqv_\w+)\s*\(", hdr, re.M))
    assert declared == set(_lib.EXPORTED)


def test_library_loads_and_exports_every_symbol():
    from paper_2511_17361_b200 import build
    if not os.path.exists(_lib.LIB_PATH):
        build.build()
    L = ctypes.CDLL(_lib.LIB_PATH)
    for sym in _lib.EXPORTED:
        assert hasattr(L, sym), sym
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    for sym in _lib.EXPORTED:
        assert re.search(rf"\bT {sym}\b", out), sym
    lib = _lib.lib()  # no device needed for these
    assert lib.sqv_abi_version() == 1
    g = P.VoxelGridSpec()._c()
    assert lib.sqv_tiles_per_frame(ctypes.byref(g)) == 25 * 25 * 1
    assert lib.sqv_workspace_bytes(4, 2000, 18, ctypes.byref(g), 10**6) > 0
    assert lib.sqv_workspace_bytes(4, 2000, 99, ctypes.byref(g), 0) == 0  # unsupported C


def test_product_has_no_oracle_dependency():
    """The product never imports, loads or links the checker (oracle/)."""
    pkg = os.path.join(ROOT, "paper_2511_17361_b200")
    pat = re.compile(r"^\s*(from\s+oracle|import\s+oracle)|sqv_oracle|libsqv_oracle|oracle/",
                     re.M)
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                assert not pat.search(open(os.path.join(dirpath, f)).read()), f


def test_superquadric_mirrors_reference_validation():
    mk = lambda **kw: P.SuperQuadric(**{**dict(mu=[0, 0, 0], scale=[1, 1, 1], rot=[2, 0, 0, 0],
                                                 opacity=0.5, logits=[0.0, 1.0], eps1=0.1,
                                                 eps2=2.5), **kw})
    sq = mk()
    assert sq.eps1 == 0.2 and sq.eps2 == 2.0 and sq.eps_clamped
    np.testing.assert_allclose(sq.rot, [1, 0, 0, 0])
    for kw, msg in [(dict(scale=[1, 0, 1]), "strictly positive"),
                    (dict(mu=[np.nan, 0, 0]), "must be finite"),
                    (dict(opacity=1.1), r"opacity must lie in \[0, 1\]"),
                    (dict(logits=[[1.0]]), "1-D"),
                    (dict(rot=[0, 0, 0, 0]), "near-zero quaternion"),
                    (dict(mu=[0, 0]), "3-vectors")]:
        with pytest.raises(ValueError, match=msg):
            mk(**kw)
    with pytest.raises(ValueError, match="free_index"):
        P.ClassTable(("a", "b"), free_index=1)
    with pytest.raises(ValueError, match="expected 2"):
        P.Scene([mk(logits=[1.0])], P.ClassTable(("a", "b")))


def test_primitive_batch_packing_and_validation_bits():
    classes = P.ClassTable(("a", "b", "c"))
    prims = [P.SuperQuadric(mu=[i, 0, 0], scale=[1, 2, 3], rot=[1, 0, 0, 0], opacity=0.1 * i,
                            logits=[i, 0, 1], eps1=1, eps2=1) for i in range(4)]
    b = P.PrimitiveBatch.from_scenes([P.Scene(prims, classes), P.Scene(prims[:2], classes)])
    assert (b.n_frames, b.n_prims, b.n_classes) == (2, 4, 3)
    np.testing.assert_array_equal(b.n_valid, [4, 2])
    np.testing.assert_array_equal(b.mu[1, 1], [1, 0, 0])
    assert not validation_bits(b).any()
    b.opacity[0, 3] = 2.0
    b.scale[1, 3] = -1.0  # beyond n_valid: ignored
    bits = validation_bits(b)
    assert bits[0, 3] == 8 and bits[1, 3] == 0
    with pytest.raises(ValueError, match="opacity"):
        b.validate()


def test_scenegen_is_seeded_and_in_bounds():
    a = gen_frames(3, 2, 100)
    b = gen_frames(3, 2, 100)
    c = gen_frames(4, 1, 100)
    for k in P.PrimitiveBatch.FIELDS:
        np.testing.assert_array_equal(getattr(a, k), getattr(b, k))
    # frame f of seed s is frame 0 of seed s+f
    np.testing.assert_array_equal(a.mu[1], c.mu[0])
    assert np.all(a.mu[..., 0] >= -40) and np.all(a.mu[..., 0] <= 40)
    assert np.all((a.scale >= 0.2) & (a.scale <= 4.0))
    np.testing.assert_allclose(np.linalg.norm(a.rot, axis=-1), 1.0)


def test_spec_types_validate():
    with pytest.raises(ValueError):
        P.VoxelGridSpec(dims=(0, 1, 1))
    with pytest.raises(ValueError):
        P.VoxelGridSpec(resolution=0.0)
    with pytest.raises(ValueError):
        P.VoxelizeConfig(tau=-1)
    with pytest.raises(ValueError):
        P.VoxelizeConfig(semantic_mode="max")
    assert P.VoxelizeConfig().tau == 0.01 and P.VoxelGridSpec().dims == (200, 200, 16)


def test_product_fails_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(RuntimeError, match="CUDA"):
        P.Voxelizer()


def test_shard_frames_partitions():
    for n in (0, 1, 7, 6019):
        for w in (1, 2, 3, 8):
            parts = [shard_frames(n, r, w) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1


def test_iou_folds():
    # SPEC.md:502 2x2x1 example through the count folds: C=1, free index 1
    cm = np.zeros((2, 2), np.int64)
    cm[1, 0] = 1   # gt free, pred occ (0,0)
    cm[0, 0] = 1   # both occ (1,0)
    cm[0, 1] = 1   # gt occ, pred free (1,1)
    cm[1, 1] = 1
    assert abs(M.iou_from_confusion(cm) - 1 / 3) < 1e-15
    assert M.iou_from_confusion(np.diag([0, 0, 5])) == 1.0   # both empty
    per, m, valid = M.miou_from_confusion(np.diag([3, 0, 4]))
    assert m == 1.0 and list(valid) == [True, False]


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from oracle import oracle as O
    from paper_2511_17361_b200.distributed import allreduce_confusion, shard_frames
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    rng = np.random.default_rng(0)
    pred = rng.integers(0, 6, size=(9, 500)).astype(np.uint8)
    gt = rng.integers(0, 6, size=(9, 500)).astype(np.uint8)
    a, b = shard_frames(9, rank, world)
    cm = torch.from_numpy(O.confusion(pred[a:b], gt[a:b], 5).copy())
    allreduce_confusion(cm)
    if rank == 0:
        q.put((cm.numpy(), O.confusion(pred, gt, 5)))
    dist.destroy_process_group()


def test_confusion_allreduce_gloo_world2():
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, want = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    np.testing.assert_array_equal(got, want)


def test_torch_ops_registered_with_fake_shapes():
    """torch.ops.sqocc.{voxelize, prep_bin, confusion}: schemas
    and fake (meta) shapes on CPU; the real kernels need CUDA (no fallback)."""
    import torch
    from paper_2511_17361_b200 import torch_ops  # noqa: F401
    from torch._subclasses.fake_tensor import FakeTensorMode
    from torch.fx.experimental.symbolic_shapes import ShapeEnv
    F, N, C = 2, 5, 18
    m = lambda *s: torch.empty(s, dtype=torch.float64, device="meta")  # noqa: E731
    lab, vo, vc = torch.ops.sqocc.voxelize(m(F, N, 3), m(F, N, 3), m(F, N, 4), m(F, N), m(F, N, 2),
                                          m(F, N, C), [-40.0, -40.0, -1.0], [200, 200, 16], 0.4)
    assert lab.shape == (F, 16, 200, 200) and lab.dtype == torch.uint8
    assert vo.shape == (F, 16, 200, 200) and vc.shape == (F, 16, 200, 200, C)
    u8 = torch.empty(10, dtype=torch.uint8, device="meta")
    cm = torch.ops.sqocc.confusion(u8, u8, C)
    assert cm.shape == (C + 1, C + 1) and cm.dtype == torch.int64
    with FakeTensorMode(shape_env=ShapeEnv()):
        f = lambda *s: torch.empty(s, dtype=torch.float64)  # noqa: E731
        w, to, ids, n = torch.ops.sqocc.prep_bin(f(F, N, 3), f(F, N, 3), f(F, N, 4), f(F, N),
                                                 f(F, N, 2), f(F, N, C), [-40.0, -40.0, -1.0],
                                                 [200, 200, 16], 0.4)
        assert w.shape == (F, N, 6) and to.shape == (F * 625 + 1,) and n.shape == ()
    z = lambda *s: torch.zeros(s, dtype=torch.float64)  # noqa: E731
    with pytest.raises(RuntimeError):
        torch.ops.sqocc.voxelize(z(F, N, 3), z(F, N, 3), z(F, N, 4), z(F, N), z(F, N, 2),
                                 z(F, N, C), [-40.0, -40.0, -1.0], [200, 200, 16], 0.4)


def test_parity_rules_scale_with_the_term_magnitude():
    """tests/parity.py: the v_c check and the near-tie rule scale with the
    class term magnitude sum_i w_i |c_ik| when the oracle supplies it, so a
    class sum that cancels (v_c ~ 0 from large opposite terms) is judged
    against its terms, not against itself."""
    import parity as PR
    tau = 0.01
    ref_vo = np.array([[6.9e-5, 0.5]])
    ref_vc = np.array([[[-1.65e-5], [0.3]]])          # voxel 0 cancels: |v_c| << terms
    vc_abs = np.array([[[4.0e-4], [0.3]]])           # sum_i w_i |c_i|
    s0 = PR.weight_scale(ref_vo, ref_vc, tau)
    s1 = PR.weight_scale(ref_vo, ref_vc, tau, vc_abs)
    np.testing.assert_allclose(s0, [6.9e-5, 0.5])
    np.testing.assert_allclose(s1, [4.0e-4, 0.5])
    # an error of 1.6e-9 on the cancelling sum: 2.3e-5 of the lower bound
    # (fails 2e-5), 4e-6 of the term magnitude (passes)
    gpu = {"v_o": ref_vo.astype(np.float32), "v_c": ref_vc + np.array([[[1.6e-9], [0.0]]]),
           "labels": np.array([[0, 0]], np.uint8)}
    ref = {"v_o": ref_vo, "v_c": ref_vc, "labels": np.array([[0, 0]], np.uint8)}
    with pytest.raises(AssertionError, match="v_c worst"):
        PR.assert_parity(gpu, ref, tau, free_code=1, min_agreement=0.0)
    PR.assert_parity(gpu, dict(ref, v_c_abs=vc_abs), tau, free_code=1, min_agreement=0.0)
    # near-tie rule: a 2-class voxel may flip only when its top-2 gap is
    # below 1e-5 of its scale (3e-5 here, 2e-3 with the term magnitude)
    vc2 = np.array([[[2.0e-5, 2.0e-5 - 1e-10]]])
    lab = PR.label_check(np.array([[1]], np.uint8), np.array([[0]], np.uint8),
                         np.array([[3e-5]]), vc2, tau, free_code=2)
    assert lab["n_unexplained"] == 0
    vc3 = np.array([[[2.0e-5, 2.0e-5 - 1e-8]]])
    lab = PR.label_check(np.array([[1]], np.uint8), np.array([[0]], np.uint8),
                         np.array([[3e-5]]), vc3, tau, free_code=2)
    assert lab["n_unexplained"] == 1
    lab = PR.label_check(np.array([[1]], np.uint8), np.array([[0]], np.uint8),
                         np.array([[3e-5]]), vc3, tau, free_code=2,
                         ref_vc_abs=np.array([[[2e-3, 2e-3]]]))
    assert lab["n_unexplained"] == 0
