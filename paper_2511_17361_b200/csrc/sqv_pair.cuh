// sqv_pair.cuh — the per-(primitive, voxel column) weight evaluation shared by
// both tile evaluators (FFMA accumulation and tcgen05 accumulation).
#pragma once

#include "sqv_common.cuh"

namespace sqv {

constexpr int kVPT = 4;  // voxels per thread: a 1x1x4 z-column

// Local coordinates of a thread's 4 voxels for one primitive, and which of
// them are live (inside the window and not culled).
struct ColCoords {
  float p0[kVPT], p1[kVPT], p2[kVPT];
  bool live[kVPT];
};

// Can primitive R contribute to the warp's 4x4x8 voxel block at (bx0, by0,
// bz0)?  Window overlap, then a conservative geometric test: the block's
// centre in local coordinates minus its local half extent must come within
// mcut on every axis (else max|x'| > mcut on the whole block, F > kFCut).
// Evaluated lane-parallel (one primitive per lane) when building the masks.
__device__ __forceinline__ bool block_may_hit(const PrimRec& R, int bx0, int by0, int bz0) {
  if (bx0 + 3 < R.lo[0] || bx0 > R.hi[0] || by0 + 3 < R.lo[1] || by0 > R.hi[1] ||
      bz0 + 7 < R.lo[2] || bz0 > R.hi[2])
    return false;
  const float kx = (float)bx0 + 1.5f - R.cx, ky = (float)by0 + 1.5f - R.cy,
              kz = (float)bz0 + 3.5f - R.cz;
  float dmax = -1.0f, slack = 0.0f;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const float ex = R.H[3 * r] + R.L[3 * r], ey = R.H[3 * r + 1] + R.L[3 * r + 1],
                ez = R.H[3 * r + 2] + R.L[3 * r + 2];
    const float c = fmaf(kz, ez, fmaf(ky, ey, fmaf(kx, ex, R.Gh[r] + R.Gl[r])));
    const float h = 1.5f * fabsf(ex) + 1.5f * fabsf(ey) + 3.5f * fabsf(ez);
    dmax = fmaxf(dmax, fabsf(c) - h);
    slack += fabsf(c) + h;
  }
  return dmax <= R.mcut + 1e-4f * slack;
}

// Is the warp's whole 4x4x8 block inside R's window?  Then no voxel of the
// block needs the per-voxel window test (pair_coords<.., LIVE = false>).
__device__ __forceinline__ bool block_inside(const PrimRec& R, int bx0, int by0, int bz0) {
  return (bx0 >= R.lo[0]) & (bx0 + 3 <= R.hi[0]) & (by0 >= R.lo[1]) & (by0 + 3 <= R.hi[1]) &
         (bz0 >= R.lo[2]) & (bz0 + 7 <= R.hi[2]);
}

// Coordinates + liveness of primitive R at voxels (x, y, z0 + v), v < 4.
// The caller has already established — per warp, with block_may_hit — that
// the primitive can reach the warp's block, so there is no further cull
// here: a voxel is live when it is inside the window; voxels with
// F >= kFCut get w = 0 from the field itself (exactly what culling would
// have produced).
//
// Local coordinates use the exact lattice stepping of prep's split_row: the
// hi parts (10 significant bits per row, the reference offset on the same
// quantum) times small integer offsets sum exactly in FP32, the lo parts are
// small, so x' carries no cancellation error even for thin, rotated
// primitives far from their centre voxel.
template <bool EXACT_STEP, bool LIVE = true>
__device__ __forceinline__ void pair_coords(const PrimRec& R, int x, int y, int z0,
                                            ColCoords& cd) {
  // bitwise (not short-circuit) tests: no divergent branches on loaded bounds
  const bool in_xy = (x >= R.lo[0]) & (x <= R.hi[0]) & (y >= R.lo[1]) & (y <= R.hi[1]);
  const float fx = (float)x - R.cx, fy = (float)y - R.cy, fz = (float)z0 - R.cz;
  const float h0 = fmaf(fz, R.H[2], fmaf(fy, R.H[1], fmaf(fx, R.H[0], R.Gh[0])));
  const float h1 = fmaf(fz, R.H[5], fmaf(fy, R.H[4], fmaf(fx, R.H[3], R.Gh[1])));
  const float h2 = fmaf(fz, R.H[8], fmaf(fy, R.H[7], fmaf(fx, R.H[6], R.Gh[2])));
  const float l0 = fmaf(fz, R.L[2], fmaf(fy, R.L[1], fmaf(fx, R.L[0], R.Gl[0])));
  const float l1 = fmaf(fz, R.L[5], fmaf(fy, R.L[4], fmaf(fx, R.L[3], R.Gl[1])));
  const float l2 = fmaf(fz, R.L[8], fmaf(fy, R.L[7], fmaf(fx, R.L[6], R.Gl[2])));
  const int loz = R.lo[2], hiz = R.hi[2];
  cd.p0[0] = h0 + l0;
  cd.p1[0] = h1 + l1;
  cd.p2[0] = h2 + l2;
#pragma unroll
  for (int v = 1; v < kVPT; ++v) {
    const float fv = (float)v;
    if (EXACT_STEP) {  // strict: hi/lo stepping, exact
      cd.p0[v] = fmaf(fv, R.H[2], h0) + fmaf(fv, R.L[2], l0);
      cd.p1[v] = fmaf(fv, R.H[5], h1) + fmaf(fv, R.L[5], l1);
      cd.p2[v] = fmaf(fv, R.H[8], h2) + fmaf(fv, R.L[8], l2);
    } else {  // fast: <= 3 steps of the once-rounded z step (error <= 3 ulp(dz))
      cd.p0[v] = fmaf(fv, R.Ez[0], cd.p0[0]);
      cd.p1[v] = fmaf(fv, R.Ez[1], cd.p1[0]);
      cd.p2[v] = fmaf(fv, R.Ez[2], cd.p2[0]);
    }
  }
#pragma unroll
  for (int v = 0; v < kVPT; ++v) {
    const int z = z0 + v;
    cd.live[v] = LIVE ? (in_xy & (z >= loz) & (z <= hiz)) : true;
  }
}

// Field of one voxel with either SFU logs (ACC = false) or FMA-pipe ~1 ulp
// logs for the coordinates (ACC = true).  Same log-sum-exp form as field_F7.
template <bool ACC>
__device__ __forceinline__ float field_lse(float x0, float x1, float x2, float a, float b,
                                           float c) {
  const float lx = ACC ? log2_acc(fabsf(x0)) : lg2(fabsf(x0));
  const float ly = ACC ? log2_acc(fabsf(x1)) : lg2(fabsf(x1));
  const float lz = ACC ? log2_acc(fabsf(x2)) : lg2(fabsf(x2));
  const float ux = a * lx, uy = a * ly;
  const float umax = fmaxf(ux, uy);
  const float d = fmaxf(fminf(ux, uy) - umax, -126.0f);
  const float Sb = ex2(b * (umax + log2_1p_poly(ex2(d))));
  const float Z = ex2(c * lz);
  return Sb + Z;
}

template <int FIELD, bool ACC>
__device__ __forceinline__ float field_of(float x0, float x1, float x2, float a, float b,
                                          float c) {
  if (FIELD == 9) return field_F(x0, x1, x2, a, b, c);
  if (FIELD == 8) return field_F8(x0, x1, x2, a, b, c);
  return field_lse<ACC>(x0, x1, x2, a, b, c);
}

// Strict mode (FIELD 6) takes the accurate logs for primitives whose exponent
// amplifies the log error: 2/eps1 = c > 3.
template <int FIELD>
__device__ __forceinline__ bool wants_acc(const PrimRec& R) {
  return FIELD == 6 && R.c > 3.0f;
}

// The log-sum-exp field written step by step across the 4 voxels of the
// column, so the 4 independent chains are interleaved in program order (the
// evaluator is latency-bound; this is the schedule we want from ptxas).
template <bool ACC>
__device__ __forceinline__ void weights_lse4(const PrimRec& R, const ColCoords& cd,
                                             float (&w)[kVPT]) {
  const float a = R.a, b = R.b, c = R.c;
  float ux[kVPT], uy[kVPT], uz[kVPT], um[kVPT], t[kVPT], F[kVPT];
#pragma unroll
  for (int v = 0; v < kVPT; ++v) {
    ux[v] = a * (ACC ? log2_acc(fabsf(cd.p0[v])) : lg2(fabsf(cd.p0[v])));
    uy[v] = a * (ACC ? log2_acc(fabsf(cd.p1[v])) : lg2(fabsf(cd.p1[v])));
    uz[v] = c * (ACC ? log2_acc(fabsf(cd.p2[v])) : lg2(fabsf(cd.p2[v])));
  }
#pragma unroll
  for (int v = 0; v < kVPT; ++v) {
    um[v] = fmaxf(ux[v], uy[v]);
    t[v] = ex2(fmaxf(fminf(ux[v], uy[v]) - um[v], -126.0f));
  }
#pragma unroll
  for (int v = 0; v < kVPT; ++v) t[v] = log2_1p_poly(t[v]);
#pragma unroll
  for (int v = 0; v < kVPT; ++v) F[v] = ex2(b * (um[v] + t[v])) + ex2(uz[v]);
#pragma unroll
  for (int v = 0; v < kVPT; ++v)
    w[v] = (cd.live[v] & (F[v] < kFCut)) ? ex2(-F[v] * kLog2e) : 0.0f;
}

template <int FIELD, bool ACC>
__device__ __forceinline__ void weights_one(const PrimRec& R, const ColCoords& cd,
                                            float (&w)[kVPT]) {
  if (FIELD == 6 || FIELD == 7) {
    weights_lse4<ACC>(R, cd, w);
    return;
  }
#pragma unroll
  for (int v = 0; v < kVPT; ++v) {
    const float F = field_of<FIELD, ACC>(cd.p0[v], cd.p1[v], cd.p2[v], R.a, R.b, R.c);
    w[v] = (cd.live[v] && F < kFCut) ? ex2(-F * kLog2e) : 0.0f;
  }
}

// w = exp(-F) (0 for dead voxels) of one primitive.
template <int FIELD>
__device__ __forceinline__ void pair_field(const PrimRec& R, const ColCoords& cd,
                                           float (&w)[kVPT]) {
  if (wants_acc<FIELD>(R))
    weights_one<FIELD, true>(R, cd, w);
  else
    weights_one<FIELD, false>(R, cd, w);
}

// Single-primitive convenience (coords + field).
template <int FIELD, bool LIVE = true>
__device__ __forceinline__ void pair_weights(const PrimRec& R, int x, int y, int z0,
                                             float (&w)[kVPT]) {
  ColCoords cd;
  pair_coords<FIELD == 6, LIVE>(R, x, y, z0, cd);
  pair_field<FIELD>(R, cd, w);
}

}  // namespace sqv
