// sqv_pair.cuh — the per-(primitive, voxel column) weight evaluation shared by
// both tile evaluators (FFMA accumulation and tcgen05 accumulation).
#pragma once

#include "sqv_common.cuh"

namespace sqv {

constexpr int kVPT = 4;  // voxels per thread: a 1x1x4 z-column

// Weights w[v] = exp(-F) of primitive R at voxels (x, y, z0 + v), v < 4
// (core.py:237-282).  Returns false — warp-uniformly — when no
// lane of the warp has a live voxel (outside the window, or max|x'| > mcut so
// that F > kFCut and w would be exactly 0); w is then not written.
//
// Local coordinates use the exact lattice stepping of prep's split_row: the
// hi parts (10 significant bits per row) times small integer offsets sum
// exactly in FP32, the lo parts are small, so x' carries no cancellation
// error even for thin, rotated primitives far from their centre voxel.
template <int FIELD>
__device__ __forceinline__ bool pair_weights(const PrimRec& R, int x, int y, int z0,
                                             float (&w)[kVPT]) {
  const bool in_xy = x >= R.lo[0] && x <= R.hi[0] && y >= R.lo[1] && y <= R.hi[1];
  const float fx = (float)x - R.cx, fy = (float)y - R.cy, fz = (float)z0 - R.cz;
  // column base (z0) then each voxel directly: hi parts exact, short chains
  const float h0 = fmaf(fz, R.H[2], fmaf(fy, R.H[1], fmaf(fx, R.H[0], R.Gh[0])));
  const float h1 = fmaf(fz, R.H[5], fmaf(fy, R.H[4], fmaf(fx, R.H[3], R.Gh[1])));
  const float h2 = fmaf(fz, R.H[8], fmaf(fy, R.H[7], fmaf(fx, R.H[6], R.Gh[2])));
  const float l0 = fmaf(fz, R.L[2], fmaf(fy, R.L[1], fmaf(fx, R.L[0], R.Gl[0])));
  const float l1 = fmaf(fz, R.L[5], fmaf(fy, R.L[4], fmaf(fx, R.L[3], R.Gl[1])));
  const float l2 = fmaf(fz, R.L[8], fmaf(fy, R.L[7], fmaf(fx, R.L[6], R.Gl[2])));
  const float mcut = R.mcut;
  const int loz = R.lo[2], hiz = R.hi[2];
  float p0[kVPT], p1[kVPT], p2[kVPT];
  bool live[kVPT];
  bool any = false;
#pragma unroll
  for (int v = 0; v < kVPT; ++v) {
    const float fv = (float)v;
    p0[v] = fmaf(fv, R.H[2], h0) + fmaf(fv, R.L[2], l0);
    p1[v] = fmaf(fv, R.H[5], h1) + fmaf(fv, R.L[5], l1);
    p2[v] = fmaf(fv, R.H[8], h2) + fmaf(fv, R.L[8], l2);
    const int z = z0 + v;
    const float mm = fmaxf(fmaxf(fabsf(p0[v]), fabsf(p1[v])), fabsf(p2[v]));
    live[v] = in_xy && z >= loz && z <= hiz && mm <= mcut;
    any |= live[v];
  }
  if (!__any_sync(0xffffffffu, any)) return false;
  const float a = R.a, b = R.b, c = R.c;
#pragma unroll
  for (int v = 0; v < kVPT; ++v) {
    const float F = FIELD == 7   ? field_F7(p0[v], p1[v], p2[v], a, b, c)
                    : FIELD == 6 ? field_F6(p0[v], p1[v], p2[v], a, b, c)
                    : FIELD == 8 ? field_F8(p0[v], p1[v], p2[v], a, b, c)
                                 : field_F(p0[v], p1[v], p2[v], a, b, c);
    w[v] = (live[v] && F < kFCut) ? ex2(-F * kLog2e) : 0.0f;
  }
  return true;
}

}  // namespace sqv
