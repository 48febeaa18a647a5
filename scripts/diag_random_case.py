"""Re-run one test_randomized_configurations case (GPU box, diagnostics) and
print its worst v_o / v_c errors and the worst v_c voxel's term magnitude
sum_i w_i |c_i| (FP64 oracle, the checker) — for the library SQV_LIB names.
usage: python scripts/diag_random_case.py CASE"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2511_17361_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2511_17361_b200.core import PrimitiveBatch  # noqa: E402
from paper_2511_17361_b200.scenegen import gen_frames  # noqa: E402
from parity import VO_MIN_FLOOR, VO_TAIL_FLOOR_FRAC_TAU  # noqa: E402

case = int(sys.argv[1])
rng = np.random.default_rng(1000 + case)  # the same draws as the test
dims = (int(rng.integers(5, 45)), int(rng.integers(5, 45)), int(rng.integers(3, 36)))
res = float(rng.choice([0.2, 0.37, 0.5]))
origin = tuple(float(x) for x in rng.uniform(-6, 2, 3))
C = int(rng.choice([1, 2, 5, 12, 17, 18, 19, 23, 24]))
mode = "prob-sum" if rng.random() < 0.4 else "logit-sum"
prec = "fast" if rng.random() < 0.3 else "strict"
truncate = rng.random() < 0.75
F, N = int(rng.integers(1, 4)), int(rng.integers(1, 60))
spec = P.VoxelGridSpec(origin, dims, res)
tau = float(rng.choice([0.0, 0.01, 0.2]))
cfg = P.VoxelizeConfig(tau=tau, neighborhood_radius=int(rng.integers(0, 6)), semantic_mode=mode,
                       precision=prec)
smax = float(rng.choice([1.0, 4.0]))
b = gen_frames(77 + case, F, N, C, origin=origin, dims=dims, resolution=res, smax=smax)
nv = rng.integers(0, N + 1, F).astype(np.int32)
b = PrimitiveBatch(b.mu, b.scale, b.rot, b.opacity, b.eps, b.logits, n_valid=nv)
os.environ["SQV_PERSIST"] = str(case % 2)
os.environ["SQV_STREAM"] = str((case // 2) % 2)
os.environ["SQV_BIN"] = ("radix", "frame")[(case // 4) % 2]
vox = P.Voxelizer(spec, cfg, C, truncate=truncate)
r = vox(b, dense=True)
vo = r.v_o.reshape(F, -1).cpu().numpy().astype(np.float64)
vc = r.v_c.reshape(F, -1, C).cpu().numpy().astype(np.float64)
grid = O.Grid(spec.origin, spec.dims, spec.resolution)
ref = O.voxelize(O.Prims.of(b), grid, O.Cfg(tau=tau, neighborhood_radius=cfg.neighborhood_radius,
                                            truncate=truncate, prob_sum=mode == "prob-sum",
                                            free_label=r.free_code))
floor = max(VO_TAIL_FLOOR_FRAC_TAU * tau, VO_MIN_FLOOR)
rvo = np.abs(vo - ref["v_o"]) / np.maximum(ref["v_o"], floor)
scale = np.maximum(np.maximum(np.abs(ref["v_c"]).max(-1), ref["v_o"]), floor)
rvc = np.abs(vc - ref["v_c"]).max(-1) / scale
f, v = np.unravel_index(np.argmax(rvc), rvc.shape)
print({"case": case, "dims": dims, "C": C, "mode": mode, "prec": prec, "tau": tau,
       "truncate": truncate, "worst_vo": float(rvo.max()), "worst_vc": float(rvc.max()),
       "at": (int(f), int(v)), "v_o": float(ref["v_o"][f, v]), "v_c": ref["v_c"][f, v].tolist(),
       "gpu_v_c": vc[f, v].tolist()})
