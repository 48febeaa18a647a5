"""Every evaluator variant (chunk-staged / streaming x per-item / persistent)
on a dense and a sparse batch, both precisions, C = 18 and C = 24, a
tile-ragged grid: the four variants must agree (labels up to near-ties,
v_o to the parity bound), and persistent == per-item bit for bit.
(compute-sanitizer is closed on this pool; this is the substitute check.)
usage: python scripts/variant_sweep.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2511_17361_b200 as P  # noqa: E402
from paper_2511_17361_b200.scenegen import gen_frames  # noqa: E402

spec = P.VoxelGridSpec((-10.0, -9.0, -1.0), (52, 44, 20), 0.4)
for C in (18, 24):
    for n_prims in (60, 700):
        b = gen_frames(7 + n_prims, 2, n_prims, C, origin=spec.origin, dims=spec.dims,
                       resolution=spec.resolution)
        for prec in ("strict", "fast"):
            outs = {}
            for stream in ("0", "1"):
                for persist in ("0", "1"):
                    os.environ["SQV_STREAM"], os.environ["SQV_PERSIST"] = stream, persist
                    r = P.Voxelizer(spec, P.VoxelizeConfig(precision=prec), C)(b, dense=True)
                    torch.cuda.synchronize()
                    outs[stream, persist] = (r.labels.clone(), r.v_o.clone(), r.v_c.clone())
            for stream in ("0", "1"):
                a, p = outs[stream, "0"], outs[stream, "1"]
                assert all(bool(torch.equal(x, y)) for x, y in zip(a, p)), (C, n_prims, prec, stream)
            a, s_ = outs["0", "0"], outs["1", "0"]
            rel = float(((a[1] - s_[1]).abs() / a[1].abs().clamp_min(1e-5)).max())
            agree = float((a[0] == s_[0]).double().mean())
            print(f"C={C} N={n_prims} {prec}: chunk vs stream max v_o rel {rel:.2e}, "
                  f"label agreement {agree:.6f}")
            assert rel < 4e-5 and agree > 0.9999
print("variant sweep ok")
