"""Time the reference's own NumPy density path (sqocc.core.density =
exp(-inside_outside(to_local(x))), core.py:237-282) per (primitive, voxel)
pair, as SURVEY.md §8(d) asks next to the oracle numbers.

Runs in the build container only (it imports /root/reference, which the GPU
box does not have); the result is recorded in profiles/r01_reference_numpy.txt.
usage: python scripts/ref_numpy_rate.py [n_prims] [points_per_prim]
"""
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"


def main():
    n_prims = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    per = int(sys.argv[2]) if len(sys.argv) > 2 else 36000  # ~ a config-2 window
    sys.path.insert(0, REF)
    from sqocc import core  # noqa: E402  (reference package, read-only)

    rng = np.random.default_rng(20251117)
    prims = []
    for _ in range(n_prims):
        prims.append(core.SuperQuadric(
            mu=rng.uniform(-5, 5, 3), scale=rng.uniform(0.2, 4.0, 3),
            rot=core.random_unit_quat(rng), opacity=float(rng.uniform()),
            logits=rng.standard_normal(18), eps1=float(rng.uniform(0.2, 2.0)),
            eps2=float(rng.uniform(0.2, 2.0))))
    pts = [p.mu + rng.uniform(-6, 6, (per, 3)) for p in prims]
    core.density(prims[0], pts[0][:16])  # warm-up
    t0 = time.perf_counter()
    s = 0.0
    for p, x in zip(prims, pts):
        s += float(core.density(p, x).sum())
    dt = time.perf_counter() - t0
    pairs = n_prims * per
    threads = os.environ.get("OMP_NUM_THREADS", "default")
    print(f"reference NumPy density path (sqocc.core, core.py:237-282): {pairs} pairs in "
          f"{dt:.2f} s = {1e9 * dt / pairs:.1f} ns/pair ({pairs / dt:.3e} pairs/s), "
          f"1 Python thread, NumPy {np.__version__}, OMP_NUM_THREADS={threads}, "
          f"{os.cpu_count()} host CPUs; checksum {s:.6e}")


if __name__ == "__main__":
    main()
