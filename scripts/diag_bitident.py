"""Hashes of the dense outputs for fixed inputs (configs 1-4 frames and a
persistent-mode case): run once per library build and diff the lines to
check that a change is bit-neutral.  usage: python scripts/diag_bitident.py"""
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17361_b200 as P  # noqa: E402
from paper_2511_17361_b200.scenegen import gen_frames  # noqa: E402

CASES = [
    ("config1", 256, 10, dict(), (200, 200, 16), 0.4, (-40.0, -40.0, -1.0), "strict"),
    ("config2", 2000, 10, dict(), (200, 200, 16), 0.4, (-40.0, -40.0, -1.0), "strict"),
    ("config2-fast", 2000, 4, dict(), (200, 200, 16), 0.4, (-40.0, -40.0, -1.0), "fast"),
    ("config3", 4000, 4, dict(emin=0.1), (200, 200, 16), 0.4, (-40.0, -40.0, -1.0), "strict"),
    ("config4", 8000, 1, dict(), (400, 400, 32), 0.2, (-40.0, -40.0, -1.0), "strict"),
]
for name, n, F, gen, dims, res, origin, prec in CASES:
    b = gen_frames(20251117, F, n, 18, origin=origin, dims=dims, resolution=res, **gen)
    spec = P.VoxelGridSpec(origin, dims, res)
    vox = P.Voxelizer(spec, P.VoxelizeConfig(precision=prec), 18)
    r = vox(b, dense=True)
    h = hashlib.sha256()
    for t in (r.labels, r.v_o, r.v_c):
        h.update(t.cpu().numpy().tobytes())
    print(name, h.hexdigest()[:16], flush=True)
