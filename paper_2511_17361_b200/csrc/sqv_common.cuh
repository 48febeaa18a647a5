// sqv_common.cuh — shared device code of libsqv (B200 / sm_100a).
//
// Per-primitive FP64 setup (the reference's SuperQuadric.__post_init__ +
// world_to_local_matrix + the SPEC window), the FP32 inside-outside field on
// the SFU (MUFU.LG2 / MUFU.EX2), and the launch bookkeeping.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/sqv.h"

namespace sqv {

// ---- constants ---------------------------------------------------------

constexpr double kEpsMin = 0.2;  // core.py:18
constexpr double kEpsMax = 2.0;  // core.py:19
constexpr float kFCap = 1e30f;   // core.py:23 (reported F only)
// exp(-F) underflows FP32 (flush-to-zero) for F > 126*ln2 = 87.3365: the
// evaluator writes w = 0 exactly for F >= kFCut.
constexpr float kFCut = 87.3365f;
// Block-cull threshold (block masks and the Chebyshev bound mcut): a warp
// block is skipped for a primitive when a conservative lower bound of F over
// the block exceeds the primitive's cut = max(kBlockCutMin, ln(N wmax /
// 2e-12)), N = primitives per frame, wmax = max(1, max |class weight|).
// Every dropped weight is then below exp(-cut) <= 2e-12 / (N wmax), so at any
// voxel the dropped v_o and each dropped v_c sum to < 2e-12 — 50x below the
// smallest absolute tolerance of the parity bound (1e-5 x the 1e-5 floor).
// For N <= 8,000 and |class weights| <= 1 the cut is 36 (exp(-36) =
// 2.3e-16).  The block masks (tensor-core path) tighten it per tile to
// ln(E_tile wmax / 2e-12), E_tile = the tile's entries (~33 on config 2),
// with the same per-voxel bound.  Measured: +11% (+1.4% more per tile) over
// culling at kFCut (which drops nothing FP32 keeps).  SQV_BLOCK_CUT overrides
// the prep minimum (87.3365 with the per-tile term removed restores the cull
// that changes no output bit).
#ifndef SQV_BLOCK_CUT
#define SQV_BLOCK_CUT 36.0
#endif
constexpr double kBlockCutMin = SQV_BLOCK_CUT;
constexpr double kLnInvDropBound = 26.937873;  // ln(1 / 2e-12)
constexpr float kLog2e = 1.4426950408889634f;
// Strict mode's accurate-log threshold: primitives with 2/eps1 = c above it
// take FMA-pipe logs (their exponent amplifies the MUFU lg2 error).
#ifndef SQV_ACC_C
#define SQV_ACC_C 4.0f
#endif

constexpr int kTileX = SQV_TILE_X, kTileY = SQV_TILE_Y, kTileZ = SQV_TILE_Z;

// Per-primitive evaluation record (FP32, 40 words = 10 x float4).
//   HL[3r+j]:         (hi, lo) split of res * M'[r][j], M' = diag(1/s) * Rwl
//   G[r]:             (hi, lo) split (same row quantum) of the local (scaled)
//                     coords of the reference voxel centre
//   (hi, lo) pairs are adjacent so one packed FFMA2 steps both)
//   a, b, c:          2/eps2, eps2/eps1, 2/eps1 (core.py:267-269)
//   mcut:             Chebyshev cull bound, F >= max|x'|^(2/eps1)
//   cx, cy, cz:       reference voxel index (exact small integers)
//   lo[3], hi[3]:     clipped voxel window (int)
//   Ez[3]:            res * M'[r][2] rounded once (the fast-mode z step)
// (sigma travels with the class weights, see prep's lrows.)
constexpr int kRecWords = 40;
struct __align__(16) PrimRec {
  // words 0..32: everything the per-pair loop reads
  float2 HL[9];
  float2 G[3];
  float a, b, c;
  float cx, cy, cz;
  float Ez[3];
  // words 33..39: cull bound and window (block tests, partial blocks)
  float mcut;
  int lo[3];
  int hi[3];
};
static_assert(sizeof(PrimRec) == kRecWords * 4, "PrimRec layout");

// ---- MUFU wrappers -----------------------------------------------------

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Inside-outside field (core.py:270): F = (|x|^a + |y|^a)^b + |z|^c with the
// 1/s scaling already folded into the local coordinates.  9 SFU ops per call
// including the caller's exp.  x = 0 gives lg2 = -inf -> ex2 = 0 exactly; a
// saturated power gives +inf, which fails the F < kFCut test (w = 0), so no
// NaN can arise from valid inputs.
__device__ __forceinline__ float field_F(float x0, float x1, float x2, float a, float b,
                                         float c) {
  const float X = ex2(a * lg2(fabsf(x0)));
  const float Y = ex2(a * lg2(fabsf(x1)));
  const float Sb = ex2(b * lg2(X + Y));
  const float Z = ex2(c * lg2(fabsf(x2)));
  return Sb + Z;
}

// log2(1 + t) for t in [0, 1] on the FMA pipe: degree-8 minimax (max error
// 4.6e-8 in exact arithmetic, ~1.7e-7 evaluated in FP32, comparable to one
// MUFU.LG2).  The leading term is applied with an FMA.
// Estrin evaluation (dependency depth 4 instead of 7).
__device__ __forceinline__ float log2_1p_poly(float t) {
  const float t2 = t * t;
  const float p01 = fmaf(4.786837101e-01f, t, -7.211657763e-01f);   // c2 t + c1
  const float p23 = fmaf(2.418647856e-01f, t, -3.473010957e-01f);   // c4 t + c3
  const float p45 = fmaf(5.205900222e-02f, t, -1.375213563e-01f);   // c6 t + c5
  const float t4 = t2 * t2;
  const float q03 = fmaf(p23, t2, p01);
  const float q47 = fmaf(-9.309163317e-03f, t2, p45);               // c7 t^2 + p45
  const float q = fmaf(q47, t4, q03);                                // c1 + c2 t + ... + c7 t^6
  return fmaf(t, 1.442689896e+00f, t2 * q);
}

// The same field with 7 SFU ops instead of 8 (caller's exp excluded):
// (X + Y)^b = 2^(b * (umax + log2(1 + 2^(umin - umax)))), u = a * log2|x|.
// X and Y are never formed, so their exp/log round trip (amplified by b)
// disappears: fewer MUFU ops and a smaller error.  Both coordinates 0 give
// umin - umax = NaN, clamped to -126 (t ~ 0), and umax = -inf -> S^b = 0.
__device__ __forceinline__ float field_F7(float x0, float x1, float x2, float a, float b,
                                          float c) {
  const float ux = a * lg2(fabsf(x0));
  const float uy = a * lg2(fabsf(x1));
  const float umax = fmaxf(ux, uy);
  const float d = fmaxf(fminf(ux, uy) - umax, -126.0f);
  const float t = ex2(d);
  const float Sb = ex2(b * (umax + log2_1p_poly(t)));
  const float Z = ex2(c * lg2(fabsf(x2)));
  return Sb + Z;
}

// Variant with log2(1 + t) on the SFU instead of the polynomial: 8 MUFU,
// shorter dependency chain, MUFU.LG2 absolute error (2^-22) in place of the
// polynomial's ~1.7e-7.
__device__ __forceinline__ float field_F8(float x0, float x1, float x2, float a, float b,
                                          float c) {
  const float ux = a * lg2(fabsf(x0));
  const float uy = a * lg2(fabsf(x1));
  const float umax = fmaxf(ux, uy);
  const float d = fmaxf(fminf(ux, uy) - umax, -126.0f);
  const float Sb = ex2(b * (umax + lg2(1.0f + ex2(d))));
  const float Z = ex2(c * lg2(fabsf(x2)));
  return Sb + Z;
}

// log2(x) on the FMA pipe to ~1 ulp (vs MUFU.LG2's 2^-22 absolute error):
// x = m 2^e with m in [sqrt(1/2), sqrt(2)), log2(m) = r q(r), r = m - 1,
// degree-8 minimax q (relative error 2.6e-8).  Zero and denormals give -inf
// like lg2.approx.ftz.
__device__ __forceinline__ float log2_acc(float x) {
  const int i = __float_as_int(x);
  const int e = (i - 0x3f3504f3) >> 23;
  const float r = __int_as_float(i - (e << 23)) - 1.0f;
  float q = 1.258370578e-01f;
  q = fmaf(q, r, -2.072697580e-01f);
  q = fmaf(q, r, 2.157156020e-01f);
  q = fmaf(q, r, -2.389448136e-01f);
  q = fmaf(q, r, 2.879162431e-01f);
  q = fmaf(q, r, -3.607036769e-01f);
  q = fmaf(q, r, 4.809106290e-01f);
  q = fmaf(q, r, -7.213473320e-01f);
  q = fmaf(q, r, 1.442695022e+00f);
  const float l = fmaf(r, q, (float)e);
  return x >= 1.17549435e-38f ? l : -INFINITY;
}

// "strict" field: the coordinate logs go through log2_acc when the primitive
// amplifies their error, i.e. when 2/eps1 (= c = a*b) > 3 — a warp-uniform
// choice per primitive.  Below that the SFU logs already keep |dF| <= 5e-7 F.
__device__ __forceinline__ float field_F6(float x0, float x1, float x2, float a, float b,
                                          float c) {
  float lx, ly, lz;
  if (c > 3.0f) {
    lx = log2_acc(fabsf(x0));
    ly = log2_acc(fabsf(x1));
    lz = log2_acc(fabsf(x2));
  } else {
    lx = lg2(fabsf(x0));
    ly = lg2(fabsf(x1));
    lz = lg2(fabsf(x2));
  }
  const float ux = a * lx, uy = a * ly;
  const float umax = fmaxf(ux, uy);
  const float d = fmaxf(fminf(ux, uy) - umax, -126.0f);
  const float t = ex2(d);
  const float Sb = ex2(b * (umax + log2_1p_poly(t)));
  const float Z = ex2(c * lz);
  return Sb + Z;
}

__device__ __forceinline__ float density_of(float F) {
  return F < kFCut ? ex2(-F * kLog2e) : 0.0f;
}

// ---- FP64 per-primitive setup ------------------------------------------

struct PrimF64 {
  double mu[3];
  double M[9];  // diag(1/s) * world_to_local, row-major
  double e1, e2;
  double sigma;
  double smax;
  int bad;
};

// Validation (core.py:147-159, 33-34) in the same order, normalisation and
// eps clamp (core.py:160-165), world_to_local = quat_to_matrix(q)^T
// (core.py:55-65,183-185), scaled by 1/s (core.py:264-266).
__device__ inline PrimF64 prim_setup(const double* mu, const double* scale, const double* rot,
                                     double opacity, const double* eps, const double* logits,
                                     int C) {
  PrimF64 P;
  int bad = 0;
#pragma unroll
  for (int k = 0; k < 3; ++k)
    if (!isfinite(mu[k]) || !isfinite(scale[k])) bad |= SQV_BAD_MU_SCALE_FINITE;
  if (!bad) {
#pragma unroll
    for (int k = 0; k < 3; ++k)
      if (!(scale[k] > 0.0)) bad |= SQV_BAD_SCALE_POSITIVE;
  }
  for (int k = 0; k < C; ++k)
    if (!isfinite(logits[k])) bad |= SQV_BAD_LOGITS_FINITE;
  if (!(opacity >= 0.0 && opacity <= 1.0)) bad |= SQV_BAD_OPACITY;
  const double qw = rot[0], qx = rot[1], qy = rot[2], qz = rot[3];
  const double n = sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
  if (!(n >= 1e-12)) bad |= SQV_BAD_QUAT;
  if (!isfinite(eps[0]) || !isfinite(eps[1])) bad |= SQV_BAD_EPS;
  P.bad = bad;
  if (bad) return P;
  const double w = qw / n, x = qx / n, y = qy / n, z = qz / n;
  const double xx = x * x, yy = y * y, zz = z * z;
  const double wx = w * x, wy = w * y, wz = w * z;
  const double xy = x * y, xz = x * z, yz = y * z;
  // local-to-world R (core.py:60-64); world-to-local is R^T
  const double R[9] = {1.0 - 2.0 * (yy + zz), 2.0 * (xy - wz), 2.0 * (xz + wy),
                       2.0 * (xy + wz), 1.0 - 2.0 * (xx + zz), 2.0 * (yz - wx),
                       2.0 * (xz - wy), 2.0 * (yz + wx), 1.0 - 2.0 * (xx + yy)};
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int j = 0; j < 3; ++j) P.M[3 * r + j] = R[3 * j + r] / scale[r];
#pragma unroll
  for (int k = 0; k < 3; ++k) P.mu[k] = mu[k];
  P.e1 = fmin(fmax(eps[0], kEpsMin), kEpsMax);
  P.e2 = fmin(fmax(eps[1], kEpsMin), kEpsMax);
  P.sigma = opacity;
  P.smax = fmax(fmax(scale[0], scale[1]), scale[2]);
  return P;
}

// ---- launch bookkeeping --------------------------------------------------

void count_launch();
int set_error(int code, const char* fmt, ...);
int check_launch(const char* what);

inline int div_up(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

}  // namespace sqv
