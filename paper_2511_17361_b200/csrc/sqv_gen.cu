// sqv_gen.cu — device-side seeded scene generation (SPEC.md:594-597
// gen_scene): each rank of a frame stream can create its
// primitives in HBM instead of generating them on the host and copying.
//
// Counter-based Philox4x32-10: key = seed, counter = (prim, frame lo, frame
// hi, block).  Per primitive, uniform k (k < 9: mu xyz, scale xyz, opacity,
// eps1, eps2) takes block k/2, words 2(k%2)..+1 as a 53-bit fraction; normal
// m (rot wxyz, then the C logits) is the Box-Muller pair of block 16 + m/2.
// Same distributions as the host generator (scenegen.py): mu ~ U(grid
// bounds), scale ~ U[smin, smax], rot = normalised N(0,1)^4, opacity ~ U[0,1],
// eps ~ U[emin, 2], logits ~ N(0,1).  The uniform-derived fields use explicit
// _rn arithmetic, so a host mirror reproduces them bit-for-bit; the normals go
// through FP64 log/sincospi (within a few ulp of a host libm).
#include "sqv_kernels.cuh"

namespace sqv {

namespace {

struct Philox {
  uint32_t c[4];
};

__device__ __forceinline__ void philox_round(uint32_t (&c)[4], uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t lo0 = M0 * c[0], hi0 = __umulhi(M0, c[0]);
  const uint32_t lo1 = M1 * c[2], hi1 = __umulhi(M1, c[2]);
  const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
  c[0] = n0;
  c[1] = lo1;
  c[2] = n2;
  c[3] = lo0;
}

__device__ __forceinline__ void philox10(uint32_t (&c)[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    philox_round(c, k0, k1);
  }
}

__device__ __forceinline__ double u53(uint32_t a, uint32_t b) {
  return __dmul_rn(__dadd_rn(__dmul_rn((double)(a >> 5), 67108864.0), (double)(b >> 6)),
                   1.0 / 9007199254740992.0);
}

struct GenCtx {
  uint32_t k0, k1, p, flo, fhi;
  __device__ void block(uint32_t blk, uint32_t (&c)[4]) const {
    c[0] = p;
    c[1] = flo;
    c[2] = fhi;
    c[3] = blk;
    philox10(c, k0, k1);
  }
  __device__ double uniform(int k) const {
    uint32_t c[4];
    block((uint32_t)(k >> 1), c);
    return (k & 1) ? u53(c[2], c[3]) : u53(c[0], c[1]);
  }
  // Box-Muller pair m: r = sqrt(-2 ln(1 - u1)), (r cos 2 pi u2, r sin 2 pi u2)
  __device__ void normal_pair(int m, double* z0, double* z1) const {
    uint32_t c[4];
    block(16u + (uint32_t)m, c);
    const double u1 = u53(c[0], c[1]), u2 = u53(c[2], c[3]);
    const double r = sqrt(__dmul_rn(-2.0, log(__dsub_rn(1.0, u1))));
    double s, co;
    sincospi(__dmul_rn(2.0, u2), &s, &co);
    *z0 = __dmul_rn(r, co);
    *z1 = __dmul_rn(r, s);
  }
};

__device__ __forceinline__ double in_range(double lo, double hi, double u) {
  return __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u));
}

__global__ void gen_kernel(GenArgs A) {
  const int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t FN = (int64_t)A.n_frames * A.n_prims;
  if (gi >= FN) return;
  const int64_t f = gi / A.n_prims, i = gi - f * A.n_prims;
  const uint64_t frame = (uint64_t)(A.first_frame + f);
  GenCtx g{(uint32_t)A.seed, (uint32_t)(A.seed >> 32), (uint32_t)i, (uint32_t)frame,
           (uint32_t)(frame >> 32)};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    A.mu[3 * gi + a] = in_range(A.lo[a], A.hi[a], g.uniform(a));
    A.scale[3 * gi + a] = in_range(A.smin, A.smax, g.uniform(3 + a));
  }
  A.opacity[gi] = g.uniform(6);
  A.eps[2 * gi] = in_range(A.emin, 2.0, g.uniform(7));
  A.eps[2 * gi + 1] = in_range(A.emin, 2.0, g.uniform(8));
  double q[4];
  g.normal_pair(0, &q[0], &q[1]);
  g.normal_pair(1, &q[2], &q[3]);
  const double nq = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(q[0], q[0]), __dmul_rn(q[1], q[1])),
                                   __dadd_rn(__dmul_rn(q[2], q[2]), __dmul_rn(q[3], q[3]))));
  if (nq < 1e-6) {  // probability ~1e-24: a fixed unit quaternion, no rejection loop
    q[0] = 1.0;
    q[1] = q[2] = q[3] = 0.0;
  } else {
#pragma unroll
    for (int a = 0; a < 4; ++a) q[a] = __ddiv_rn(q[a], nq);
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) A.rot[4 * gi + a] = q[a];
  double* lg = A.logits + gi * A.n_classes;
  for (int m = 0; 2 * m < A.n_classes; ++m) {
    double z0, z1;
    g.normal_pair(2 + m, &z0, &z1);
    lg[2 * m] = z0;
    if (2 * m + 1 < A.n_classes) lg[2 * m + 1] = z1;
  }
}

}  // namespace

int gen_launch(const GenArgs& A, cudaStream_t s) {
  const int64_t FN = (int64_t)A.n_frames * A.n_prims;
  if (FN <= 0) return SQV_OK;
  gen_kernel<<<(unsigned)((FN + 127) / 128), 128, 0, s>>>(A);
  count_launch();
  return check_launch("gen_kernel");
}

}  // namespace sqv
