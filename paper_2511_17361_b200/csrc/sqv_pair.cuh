// sqv_pair.cuh — the per-(primitive, voxel column) weight evaluation shared by
// both tile evaluators (FFMA accumulation and tcgen05 accumulation).
#pragma once

#include "sqv_common.cuh"

namespace sqv {

constexpr int kVPT = 4;  // voxels per thread: a 1x1x4 z-column

// Can primitive R contribute to the warp's 4x4x8 voxel block at (bx0, by0,
// bz0)?  Window overlap, then conservative geometric tests: the block's
// centre in local coordinates minus its local half extent must come within
// mcut on every axis (else max|x'| > mcut on the whole block, F > the
// primitive's cut), and the field at the nearest corner of that local box
// must be below the cut (recovered as mcut^c; see kBlockCutMin).
// Evaluated lane-parallel (one primitive per lane) when building the masks.
__device__ __forceinline__ bool block_may_hit(const PrimRec& R, int bx0, int by0, int bz0) {
  if (bx0 + 3 < R.lo[0] || bx0 > R.hi[0] || by0 + 3 < R.lo[1] || by0 > R.hi[1] ||
      bz0 + 7 < R.lo[2] || bz0 > R.hi[2])
    return false;
  const float kx = (float)bx0 + 1.5f - R.cx, ky = (float)by0 + 1.5f - R.cy,
              kz = (float)bz0 + 3.5f - R.cz;
  float dmax = -1.0f, slack = 0.0f, m[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const float ex = R.HL[3 * r].x + R.HL[3 * r].y, ey = R.HL[3 * r + 1].x + R.HL[3 * r + 1].y,
                ez = R.HL[3 * r + 2].x + R.HL[3 * r + 2].y;
    const float c = fmaf(kz, ez, fmaf(ky, ey, fmaf(kx, ex, R.G[r].x + R.G[r].y)));
    const float h = 1.5f * fabsf(ex) + 1.5f * fabsf(ey) + 3.5f * fabsf(ez);
    m[r] = fabsf(c) - h;
    dmax = fmaxf(dmax, m[r]);
    slack += fabsf(c) + h;
  }
  const float e = 1e-4f * slack;  // covers the FP32 error of c and h
  if (dmax > R.mcut + e) return false;
  // Tighter: F grows with each |x'_r|, so over the block F >= F at the
  // box corner nearest the centre, |x'_r| >= max(|c_r| - h_r, 0).  Culled
  // only with a 2% margin over the cut, far above the SFU field error, so
  // every culled pair has F > cut, i.e. w < exp(-cut).
  const float F = field_F(fmaxf(m[0] - e, 0.0f), fmaxf(m[1] - e, 0.0f), fmaxf(m[2] - e, 0.0f),
                          R.a, R.b, R.c);
  return F < 1.02f * ex2(R.c * lg2(R.mcut));  // the primitive's field threshold
}

// Is the warp's whole 4x4x8 block inside R's window?  Then no voxel of the
// block needs the per-voxel window test (pair_coords<.., LIVE = false>).
__device__ __forceinline__ bool block_inside(const PrimRec& R, int bx0, int by0, int bz0) {
  return (bx0 >= R.lo[0]) & (bx0 + 3 <= R.hi[0]) & (by0 >= R.lo[1]) & (by0 + 3 <= R.hi[1]) &
         (bz0 >= R.lo[2]) & (bz0 + 7 <= R.hi[2]);
}

// The block mask of one (tile, primitive) entry: which of the 8x8x16 tile's
// 8 warp blocks (4x4x8, bit b = (z half, y half, x half)) the primitive can
// reach (bits 0-7), which lie wholly inside its window (bits 8-15), and
// strict mode's accurate-log flag (bit 16, c > acc_c).  The cull decisions
// are block_may_hit's (window overlap, the Chebyshev box bound, the
// nearest-corner field bound, all conservative), with the shared parts
// computed once per entry (the 8 local block centres differ by fixed lattice
// steps); a block whose nearest local corner is deep inside — (2^b + 1)
// max|x'|^c well below the cut — is marked without the 8-MUFU field test.
// A "hit" that could have been culled only costs evaluation work: those
// pairs get their exact FP32 w.  rec: the primitive's record (global),
// wmax: its class-weight padding column, e_tile: the tile's entry count.
__device__ __forceinline__ uint32_t entry_block_mask(const float* rec, float wmax, int e_tile,
                                                     int tx, int ty, int tz, float acc_c) {
  PrimRec R;
  const float4* src = reinterpret_cast<const float4*>(rec);
  float4* dst = reinterpret_cast<float4*>(&R);
#pragma unroll
  for (int q = 0; q < kRecWords / 4; ++q) dst[q] = __ldg(src + q);
  const int x0 = tx * kTileX, y0 = ty * kTileY, z0 = tz * kTileZ;
  float ex[3], ey[3], ez[3], c0[3], h[3], stepx[3], stepy[3], stepz[3];
  const float kx = (float)x0 + 1.5f - R.cx, ky = (float)y0 + 1.5f - R.cy,
              kz = (float)z0 + 3.5f - R.cz;
  float span = 0.0f;  // bounds |c| + h of every block: one FP32 error margin per entry
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    ex[r] = R.HL[3 * r].x + R.HL[3 * r].y;
    ey[r] = R.HL[3 * r + 1].x + R.HL[3 * r + 1].y;
    ez[r] = R.HL[3 * r + 2].x + R.HL[3 * r + 2].y;
    c0[r] = fmaf(kz, ez[r], fmaf(ky, ey[r], fmaf(kx, ex[r], R.G[r].x + R.G[r].y)));
    h[r] = 1.5f * fabsf(ex[r]) + 1.5f * fabsf(ey[r]) + 3.5f * fabsf(ez[r]);
    stepx[r] = 4.0f * ex[r];
    stepy[r] = 4.0f * ey[r];
    stepz[r] = 8.0f * ez[r];
    span += fabsf(c0[r]) + fabsf(stepx[r]) + fabsf(stepy[r]) + fabsf(stepz[r]) + h[r];
  }
  const float eps = 1e-4f * span;  // FP32 error of c, h (incl. the stepped centres)
  const float cut = R.mcut + eps;
  // The field threshold of this (tile, primitive) entry.  At most E_tile
  // primitives reach a voxel of this tile, so cut = ln(E_tile wmax / 2e-12)
  // keeps the dropped mass per voxel < 2e-12 (wmax rides in the class-weight
  // row's padding column, written by prep; +0.01 covers __logf's error).
  // The primitive's own (N-based) threshold mcut^c is the upper limit.
  const float cut_f = fminf(ex2(R.c * lg2(R.mcut)),
                            __logf((float)e_tile * wmax) + (float)kLnInvDropBound + 0.01f);
  // window overlap / containment of the two block positions on each axis
  const int* lo = R.lo;
  const int* hi = R.hi;
  const bool wx[2] = {x0 + 3 >= lo[0] && x0 <= hi[0], x0 + 7 >= lo[0] && x0 + 4 <= hi[0]};
  const bool wy[2] = {y0 + 3 >= lo[1] && y0 <= hi[1], y0 + 7 >= lo[1] && y0 + 4 <= hi[1]};
  const bool wz[2] = {z0 + 7 >= lo[2] && z0 <= hi[2], z0 + 15 >= lo[2] && z0 + 8 <= hi[2]};
  const bool ix[2] = {x0 >= lo[0] && x0 + 3 <= hi[0], x0 + 4 >= lo[0] && x0 + 7 <= hi[0]};
  const bool iy[2] = {y0 >= lo[1] && y0 + 3 <= hi[1], y0 + 4 >= lo[1] && y0 + 7 <= hi[1]};
  const bool iz[2] = {z0 >= lo[2] && z0 + 7 <= hi[2], z0 + 8 >= lo[2] && z0 + 15 <= hi[2]};
  // sure-hit radius: (2^b + 1) M^c <= 0.5 kFCut  <=>  M <= (0.5 kFCut / (2^b + 1))^(1/c)
  const float inv_c = 1.0f / R.c;
  const float sure = ex2(inv_c * lg2(0.5f * cut_f / (ex2(R.b) + 1.0f)));
  unsigned m = 0;
#pragma unroll
  for (int bb = 0; bb < 8; ++bb) {
    const int ox = bb & 1, oy = (bb >> 1) & 1, oz = bb >> 2;
    if (!(wx[ox] && wy[oy] && wz[oz])) continue;
    float mm[3], dmax = -1.0f;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      float c = c0[r];
      if (ox) c += stepx[r];
      if (oy) c += stepy[r];
      if (oz) c += stepz[r];
      mm[r] = fabsf(c) - h[r];
      dmax = fmaxf(dmax, mm[r]);
    }
    if (dmax > cut) continue;
    bool hit = dmax <= sure;
    if (!hit) {
      const float F = field_F(fmaxf(mm[0] - eps, 0.0f), fmaxf(mm[1] - eps, 0.0f),
                              fmaxf(mm[2] - eps, 0.0f), R.a, R.b, R.c);
      hit = F < 1.02f * cut_f;
    }
    if (hit) m |= (1u << bb) | ((unsigned)(ix[ox] && iy[oy] && iz[oz]) << (8 + bb));
  }
  // strict mode: the evaluator's accurate-log list (FMA-pipe logs for c > acc_c)
  if (m && R.c > acc_c) m |= 1u << 16;
  return m;
}

// ---- packed FP32x2 helpers (FFMA2 / FADD2 / FMUL2: two lanes of work per
// issue slot; same IEEE round-to-nearest results as the scalar ops) --------
__device__ __forceinline__ float2 bc2(float s) { return make_float2(s, s); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }

// log2_1p_poly on a pair (same operations, same rounding).
__device__ __forceinline__ float2 log2_1p_poly2(float2 t) {
  const float2 t2 = mul2(t, t);
  const float2 p01 = fma2(bc2(4.786837101e-01f), t, bc2(-7.211657763e-01f));
  const float2 p23 = fma2(bc2(2.418647856e-01f), t, bc2(-3.473010957e-01f));
  const float2 p45 = fma2(bc2(5.205900222e-02f), t, bc2(-1.375213563e-01f));
  const float2 t4 = mul2(t2, t2);
  const float2 q03 = fma2(p23, t2, p01);
  const float2 q47 = fma2(bc2(-9.309163317e-03f), t2, p45);
  const float2 q = fma2(q47, t4, q03);
  return fma2(t, bc2(1.442689896e+00f), mul2(t2, q));
}

// 2^x for x in [-125, 0] on the FMA pipe, packed: n = rint(x) by the
// 1.5*2^23 shifter, f = x - n in [-0.5, 0.5] exactly, degree-6 minimax for
// 2^f (max relative error 1.0e-7 evaluated in FP32, below MUFU.EX2's), the
// exponent added as an integer.  x < -125 is clamped (callers only feed
// arguments that are zeroed or < 2^-125 anyway).
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  x = make_float2(fmaxf(x.x, -125.0f), fmaxf(x.y, -125.0f));
  const float2 j = add2(x, bc2(12582912.0f));
  const float2 n = add2(j, bc2(-12582912.0f));
  const float2 f = fma2(n, bc2(-1.0f), x);
  float2 p = bc2(1.5345809515565634e-04f);
  p = fma2(p, f, bc2(1.3399932067841291e-03f));
  p = fma2(p, f, bc2(9.618489071726799e-03f));
  p = fma2(p, f, bc2(5.550328642129898e-02f));
  p = fma2(p, f, bc2(2.4022646248340607e-01f));
  p = fma2(p, f, bc2(6.931471824645996e-01f));
  p = fma2(p, f, bc2(1.0f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(j.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(j.y) << 23)));
}

#ifndef SQV_EXP_POLY
#define SQV_EXP_POLY 0
#endif

// log2_acc on a pair: the exponent split is integer work per lane, the
// polynomial runs packed.
__device__ __forceinline__ float2 log2_acc2(float2 x) {
  const int i0 = __float_as_int(x.x), i1 = __float_as_int(x.y);
  const int e0 = (i0 - 0x3f3504f3) >> 23, e1 = (i1 - 0x3f3504f3) >> 23;
  const float2 r = add2(make_float2(__int_as_float(i0 - (e0 << 23)),
                                    __int_as_float(i1 - (e1 << 23))), bc2(-1.0f));
  float2 q = bc2(1.258370578e-01f);
  q = fma2(q, r, bc2(-2.072697580e-01f));
  q = fma2(q, r, bc2(2.157156020e-01f));
  q = fma2(q, r, bc2(-2.389448136e-01f));
  q = fma2(q, r, bc2(2.879162431e-01f));
  q = fma2(q, r, bc2(-3.607036769e-01f));
  q = fma2(q, r, bc2(4.809106290e-01f));
  q = fma2(q, r, bc2(-7.213473320e-01f));
  q = fma2(q, r, bc2(1.442695022e+00f));
  // x = 0 (or denormal) is not special-cased: it yields about -127 instead
  // of -inf, and every power built from it (c, a*b >= 1) still underflows
  // to exactly 0
  return fma2(r, q, make_float2((float)e0, (float)e1));
}

// Strict accurate-log primitives (c = 2/eps1 > SQV_ACC_C) take the log of
// the coordinate's parts (log2_acc2_hl) instead of the rounded coordinate:
// the coordinate's 0.5-ulp rounding reaches w = exp(-F) as F c 6e-8, 6.9e-6
// at the density floor (F = 11.5) for c = 10, most of the 1e-5 budget.
// Measured on 1,024 config-1 frames: worst |dv_o| / v_o 1.19e-5 -> 9.7e-6
// (the four worst voxels all sat on c = 7.5-9.7 primitives); config 2
// -1.15%, config 3 -0.85% (a Fast2Sum form of the same fold: -1.3%/-1.4%).
#ifndef SQV_ACC_PARTS
#define SQV_ACC_PARTS 1
#endif

// log2|h + l| of the coordinate's exact parts (h the lattice-exact hi sum,
// l the lo sum) rather than of its rounding s = fl(h + l): log2_acc2's
// reduction takes e from s, then r = sign(s) 2^-e h - 1 (exact, Sterbenz)
// + sign(s) 2^-e l, rounded once, so r carries the coordinate to a fraction
// of s's ulp.  s = 0 (h = -l, both small) gives r = 0 and the log's floor
// -127 like log2_acc2.
__device__ __forceinline__ float2 log2_acc2_hl(float2 s, float2 h, float2 l) {
  const int i0 = __float_as_int(s.x) & 0x7fffffff, i1 = __float_as_int(s.y) & 0x7fffffff;
  const int e0 = (i0 - 0x3f3504f3) >> 23, e1 = (i1 - 0x3f3504f3) >> 23;
  const float2 sc = make_float2(
      __int_as_float((0x3f800000 - (e0 << 23)) | (__float_as_int(s.x) & 0x80000000)),
      __int_as_float((0x3f800000 - (e1 << 23)) | (__float_as_int(s.y) & 0x80000000)));
  const float2 r = fma2(l, sc, fma2(h, sc, bc2(-1.0f)));
  float2 q = bc2(1.258370578e-01f);
  q = fma2(q, r, bc2(-2.072697580e-01f));
  q = fma2(q, r, bc2(2.157156020e-01f));
  q = fma2(q, r, bc2(-2.389448136e-01f));
  q = fma2(q, r, bc2(2.879162431e-01f));
  q = fma2(q, r, bc2(-3.607036769e-01f));
  q = fma2(q, r, bc2(4.809106290e-01f));
  q = fma2(q, r, bc2(-7.213473320e-01f));
  q = fma2(q, r, bc2(1.442695022e+00f));
  return fma2(r, q, make_float2((float)e0, (float)e1));
}

// Local coordinates of a thread's 4 voxels, packed by voxel pairs:
// P[r][h] = coordinate r of voxels (2h, 2h+1); H, L its hi and lo parts
// (strict accurate-log primitives, SQV_ACC_PARTS).
struct ColCoords2 {
  float2 P[3][2];
  float2 H[3][2], L[3][2];
  bool live[kVPT];
  int in_xy;
};

// u if voxel z of a column inside the xy window is inside [lo, hi], else
// +inf: one predicate chain per voxel (setp ... .and) and one select
__device__ __forceinline__ float live_sel(float u, int z, int lo, int hi, int in_xy) {
  float r;
  asm("{\n\t.reg .pred p;\n\t"
      "setp.ne.s32 p, %4, 0;\n\t"
      "setp.ge.and.s32 p, %1, %2, p;\n\t"
      "setp.le.and.s32 p, %1, %3, p;\n\t"
      "selp.f32 %0, %5, 0f7F800000, p;\n}"
      : "=f"(r)
      : "r"(z), "r"(lo), "r"(hi), "r"(in_xy), "f"(u));
  return r;
}

// Coordinates + liveness of primitive R at voxels (x, y, z0 + v), v < 4.
// The caller has already established — per warp, with block_may_hit — that
// the primitive can reach the warp's block, so there is no further cull
// here: a voxel is live when it is inside the window (LIVE = false: the
// caller knows the whole block is); voxels with F >= kFCut get w = 0 from the
// field itself (exactly what culling would have produced).
//
// Local coordinates use the exact lattice stepping of prep's split_row: the
// hi parts (10 significant bits per row, the reference offset on the same
// quantum) times small integer offsets sum exactly in FP32, the lo parts are
// small, so x' carries no cancellation error even for thin, rotated
// primitives far from their centre voxel.  (hi, lo) run as one packed pair.
template <bool EXACT_STEP, bool LIVE = true, bool PARTS = false>
__device__ __forceinline__ void pair_coords(const PrimRec& R, int x, int y, int z0,
                                            ColCoords2& cd) {
  const float fx = (float)x - R.cx, fy = (float)y - R.cy, fz = (float)z0 - R.cz;
  const float2 v01 = make_float2(0.0f, 1.0f), v23 = make_float2(2.0f, 3.0f);
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    // (h, l) = (hi, lo) parts of coordinate r at voxel 0
    const float2 hl =
        fma2(bc2(fz), R.HL[3 * r + 2], fma2(bc2(fy), R.HL[3 * r + 1], fma2(bc2(fx), R.HL[3 * r], R.G[r])));
    if (EXACT_STEP) {  // strict: hi/lo stepping, exact
      const float2 h01 = fma2(v01, bc2(R.HL[3 * r + 2].x), bc2(hl.x));
      const float2 h23 = fma2(v23, bc2(R.HL[3 * r + 2].x), bc2(hl.x));
      const float2 l01 = fma2(v01, bc2(R.HL[3 * r + 2].y), bc2(hl.y));
      const float2 l23 = fma2(v23, bc2(R.HL[3 * r + 2].y), bc2(hl.y));
      cd.P[r][0] = add2(h01, l01);
      cd.P[r][1] = add2(h23, l23);
      if (PARTS) {  // the exact parts, for log2_acc2_hl
        cd.H[r][0] = h01;
        cd.H[r][1] = h23;
        cd.L[r][0] = l01;
        cd.L[r][1] = l23;
      }
    } else {  // fast: <= 3 steps of the once-rounded z step (error <= 3 ulp(dz))
      const float p0 = hl.x + hl.y;
      cd.P[r][0] = fma2(v01, bc2(R.Ez[r]), bc2(p0));
      cd.P[r][1] = fma2(v23, bc2(R.Ez[r]), bc2(p0));
    }
  }
  if (LIVE) {
    // bitwise (not short-circuit) tests: no divergent branches on loaded bounds
    const bool in_xy = (x >= R.lo[0]) & (x <= R.hi[0]) & (y >= R.lo[1]) & (y <= R.hi[1]);
    const int loz = R.lo[2], hiz = R.hi[2];
    cd.in_xy = in_xy;
#pragma unroll
    for (int v = 0; v < kVPT; ++v) {
      const int z = z0 + v;
      cd.live[v] = in_xy & (z >= loz) & (z <= hiz);
    }
  } else {
#pragma unroll
    for (int v = 0; v < kVPT; ++v) cd.live[v] = true;
  }
}

__device__ __forceinline__ float2 abs2(float2 a) { return make_float2(fabsf(a.x), fabsf(a.y)); }

template <bool ACC>
__device__ __forceinline__ float2 log2p(float2 a) {
  if (ACC) return log2_acc2(abs2(a));
  return make_float2(lg2(fabsf(a.x)), lg2(fabsf(a.y)));
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
// amplifies the log error: 2/eps1 = c > SQV_ACC_C (sqv_common.cuh).
template <int FIELD>
__device__ __forceinline__ bool wants_acc(const PrimRec& R) {
  return FIELD == 6 && R.c > SQV_ACC_C;
}

// The log-sum-exp field of the column's 4 voxels as two packed voxel pairs:
// the FMA-pipe work (scalings, the log2(1+t) polynomial, sums) issues once
// per pair, the SFU work per voxel.  Split in two stages so the evaluator can
// software-pipeline primitives (stage_logs of the next primitive interleaves
// with stage_exps of the current one); PairState is the hand-off.
constexpr float kLog2Log2e = 0.52876637294479f;  // log2(log2(e))

struct PairState {
  float2 um[2], uz[2], t[2];
  float b, cw;
};

// Stage 1: coordinates, the three logs, umax and t = 2^(umin - umax).  Dead
// voxels (outside the window) get uz = +inf: Z = F = inf and w = 0.
template <bool EXACT_STEP, bool LIVE, bool ACC>
__device__ __forceinline__ void stage_logs(const PrimRec& R, int x, int y, int z0,
                                           PairState& S) {
  constexpr bool kParts = SQV_ACC_PARTS && EXACT_STEP && ACC;
  ColCoords2 cd;
  pair_coords<EXACT_STEP, LIVE, kParts>(R, x, y, z0, cd);
  const float a = R.a, c = R.c;
  auto lg = [&](int r, int h) {
    return kParts ? log2_acc2_hl(cd.P[r][h], cd.H[r][h], cd.L[r][h]) : log2p<ACC>(cd.P[r][h]);
  };
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const float2 ux = mul2(bc2(a), lg(0, h));
    const float2 uy = mul2(bc2(a), lg(1, h));
    // log2(log2 e) folded into the exponents (2^(u + k) = log2(e) 2^u; see
    // stage_exps)
    float2 uz = fma2(bc2(c), lg(2, h), bc2(kLog2Log2e));
    // umin - umax = -|ux - uy| (the same rounded value); both coordinates 0
    // give NaN, clamped to -126 (t ~ 0) while umax = -inf makes S^b = 0
    S.um[h] = make_float2(fmaxf(ux.x, uy.x), fmaxf(ux.y, uy.y));
    const float2 dd = add2(ux, make_float2(-uy.x, -uy.y));
    const float2 d = make_float2(fmaxf(-fabsf(dd.x), -126.0f), fmaxf(-fabsf(dd.y), -126.0f));
    // fast mode takes one voxel pair's t on the FMA pipe (+1.4%: the SFU
    // binds there; strict, whose accurate logs load the FMA pipe, is neutral
    // with it and -1.1% with both pairs' t there, so it keeps the SFU)
    if (SQV_EXP_POLY >= 2 || (!EXACT_STEP && h == 0))
      S.t[h] = ex2_poly2(d);
    else
      S.t[h] = make_float2(ex2(d.x), ex2(d.y));
    if (LIVE) {
      if (EXACT_STEP) {  // strict: one predicate chain per voxel (+0.4%; fast: -0.2%)
        uz.x = live_sel(uz.x, z0 + 2 * h, R.lo[2], R.hi[2], cd.in_xy);
        uz.y = live_sel(uz.y, z0 + 2 * h + 1, R.lo[2], R.hi[2], cd.in_xy);
      } else {
        uz.x = cd.live[2 * h] ? uz.x : INFINITY;
        uz.y = cd.live[2 * h + 1] ? uz.y : INFINITY;
      }
    }
    S.uz[h] = uz;
  }
  S.b = R.b;
}

// Stage 2: log2(1 + t), S^b, Z, F and w = exp(-F).  w = 0 exactly once
// -F log2(e) < -126 (ftz), i.e. for every F > kFCut — the same zero the block
// cull assumes — so no select is needed (F is never NaN: see above).
// FOLD (paired with stage_logs, which folds k into uz): the exponents carry
// k = log2(log2 e), so F log2(e) = 2^(e + k) + 2^(uz + k) needs no scaling
// multiply (fast: +0.7% and max |dv_o|/v_o 1.1e-5 -> 1.0e-5; strict: -0.9%
// in the round-1 chunk-staged kernel, +0.7% config 2 / +0.6% config 3 in
// the streaming one, worst config-1 |dv_o|/v_o 9.0e-6 -> 7.6e-6).
template <bool FOLD>
__device__ __forceinline__ void stage_exps(const PairState& S, float (&w)[kVPT]) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const float2 l1p = log2_1p_poly2(S.t[h]);
    float2 F, arg;
    if (FOLD) {
      const float2 e = fma2(bc2(S.b), add2(S.um[h], l1p), bc2(kLog2Log2e));
      const float2 Fl = add2(make_float2(ex2(e.x), ex2(e.y)), make_float2(ex2(S.uz[h].x), ex2(S.uz[h].y)));
      F = mul2(Fl, bc2(1.0f / kLog2e));  // only for the polynomial exp below
      arg = make_float2(-Fl.x, -Fl.y);
    } else {
      const float2 e = mul2(bc2(S.b), add2(S.um[h], l1p));
      F = add2(make_float2(ex2(e.x), ex2(e.y)), make_float2(ex2(S.uz[h].x), ex2(S.uz[h].y)));
      arg = mul2(F, bc2(-kLog2e));
    }
    if (SQV_EXP_POLY >= 1) {
      const float2 v = ex2_poly2(arg);
      w[2 * h] = F.x < kFCut ? v.x : 0.0f;
      w[2 * h + 1] = F.y < kFCut ? v.y : 0.0f;
    } else {
      w[2 * h] = ex2(arg.x);
      w[2 * h + 1] = ex2(arg.y);
    }
  }
}

template <int FIELD, bool ACC>
__device__ __forceinline__ void weights_one(const PrimRec& R, const ColCoords2& cd,
                                            float (&w)[kVPT]) {
#pragma unroll
  for (int v = 0; v < kVPT; ++v) {
    const float x0 = (v & 1) ? cd.P[0][v >> 1].y : cd.P[0][v >> 1].x;
    const float x1 = (v & 1) ? cd.P[1][v >> 1].y : cd.P[1][v >> 1].x;
    const float x2 = (v & 1) ? cd.P[2][v >> 1].y : cd.P[2][v >> 1].x;
    const float F = field_of<FIELD, ACC>(x0, x1, x2, R.a, R.b, R.c);
    w[v] = (cd.live[v] && F < kFCut) ? ex2(-F * kLog2e) : 0.0f;
  }
}

// w = exp(-F) (0 for dead voxels) of one primitive.
template <int FIELD>
__device__ __forceinline__ void pair_field(const PrimRec& R, const ColCoords2& cd,
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
  if (FIELD == 6 || FIELD == 7) {
    PairState S;
    if (wants_acc<FIELD>(R))
      stage_logs<FIELD == 6, LIVE, true>(R, x, y, z0, S);
    else
      stage_logs<FIELD == 6, LIVE, false>(R, x, y, z0, S);
    stage_exps<true>(S, w);
    return;
  }
  ColCoords2 cd;
  pair_coords<false, LIVE>(R, x, y, z0, cd);
  pair_field<FIELD>(R, cd, w);
}

}  // namespace sqv
