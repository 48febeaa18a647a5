"""Host mirror of the device scene generator (csrc/sqv_gen.cu) for tests:
Philox4x32-10 in NumPy and the same per-field formulas.  Uniform-derived
fields are reproduced bit-for-bit; normals (FP64 log/sincospi on the device)
to a few ulp."""
import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK = np.uint64(0xFFFFFFFF)


def philox10(c, k0, k1):
    c = [np.asarray(x, np.uint64) & MASK for x in c]
    k0, k1 = int(k0), int(k1)
    for r in range(10):
        if r:
            k0 = (k0 + W0) & 0xFFFFFFFF
            k1 = (k1 + W1) & 0xFFFFFFFF
        p0 = M0 * c[0]
        p1 = M1 * c[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK
        c = [hi1 ^ c[1] ^ np.uint64(k0), lo1, hi0 ^ c[3] ^ np.uint64(k1), lo0]
    return c


def u53(a, b):
    return ((a >> np.uint64(5)).astype(np.float64) * 67108864.0
            + (b >> np.uint64(6)).astype(np.float64)) * (1.0 / 9007199254740992.0)


def gen(seed, n_frames, n_prims, n_classes, lo, hi, smin, smax, emin, first_frame=0):
    F, N, C = n_frames, n_prims, n_classes
    f = np.arange(F, dtype=np.uint64)[:, None] + np.uint64(first_frame)
    i = np.arange(N, dtype=np.uint64)[None, :]
    f, i = np.broadcast_arrays(f, i)
    k0, k1 = seed & 0xFFFFFFFF, seed >> 32

    def block(b):
        return philox10([i, f & MASK, f >> np.uint64(32), np.full_like(i, b)], k0, k1)

    def uniform(k):
        c = block(k >> 1)
        return u53(c[2], c[3]) if k & 1 else u53(c[0], c[1])

    def normal_pair(m):
        c = block(16 + m)
        u1, u2 = u53(c[0], c[1]), u53(c[2], c[3])
        r = np.sqrt(-2.0 * np.log(1.0 - u1))
        return r * np.cos(np.pi * (2.0 * u2)), r * np.sin(np.pi * (2.0 * u2))

    rng = lambda a, b, u: a + (b - a) * u
    mu = np.stack([rng(lo[a], hi[a], uniform(a)) for a in range(3)], -1)
    scale = np.stack([rng(smin, smax, uniform(3 + a)) for a in range(3)], -1)
    opacity = uniform(6)
    eps = np.stack([rng(emin, 2.0, uniform(7)), rng(emin, 2.0, uniform(8))], -1)
    q = np.stack([*normal_pair(0), *normal_pair(1)], -1)
    nq = np.sqrt((q[..., 0] * q[..., 0] + q[..., 1] * q[..., 1])
                 + (q[..., 2] * q[..., 2] + q[..., 3] * q[..., 3]))
    rot = q / nq[..., None]
    lg = []
    for m in range((C + 1) // 2):
        z0, z1 = normal_pair(2 + m)
        lg += [z0, z1]
    logits = np.stack(lg[:C], -1)
    return mu, scale, rot, opacity, eps, logits
