// sqv_prep.cu — K1 per-primitive preparation and K3 bin emission.
//
// K1 (one thread per (frame, primitive), FP64): validation, quaternion
// normalisation, eps clamp (core.py:143-173), scaled world->local matrix
// (core.py:183-185, 264-266), the SPEC voxel window (ledger
// SPEC.md:382) evaluated with the same IEEE expressions as the oracle, the
// overlapped-tile count, and the FP32 evaluation record (PrimRec) the tile
// evaluator consumes.
//
// K3 (one thread per primitive): writes one (tile key, primitive) entry per
// overlapped tile, in primitive order, and counts entries per tile.
#include "sqv_common.cuh"
#include "sqv_kernels.cuh"

namespace sqv {

// Split v (FP64) into hi + lo where every hi of the row is a multiple of the
// row quantum q (10 significant bits of the row's largest entry).  Then
// k * hi is exact for |k| < 2^12 and the sum of the three hi products of a
// row is exact in FP32, so lattice offsets never cancel catastrophically.
// The reference-voxel offset g of the row is split on the same quantum, so
// g_hi + sum_j k_j * hi_j is an exact FP32 sum too.
__device__ inline void split_row(const double v[3], double g, float2 hl[3], float2* gp) {
  const double m = fmax(fmax(fabs(v[0]), fabs(v[1])), fabs(v[2]));
  if (m == 0.0) {
#pragma unroll
    for (int j = 0; j < 3; ++j) hl[j] = make_float2(0.0f, 0.0f);
    *gp = make_float2(0.0f, (float)g);
    return;
  }
  int e;
  frexp(m, &e);                       // m in [2^(e-1), 2^e)
  const double q = ldexp(1.0, e - 10);
  const double iq = ldexp(1.0, 10 - e);
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const double h = rint(v[j] * iq) * q;
    hl[j] = make_float2((float)h,     // exact: <= 11 significant bits
                        (float)(v[j] - h));
  }
  const double gh = rint(g * iq) * q;
  *gp = make_float2((float)gh,        // exact while |g| < 2^(e+13)
                    (float)(g - gh));
}

// Primitive gi of the batch: validation, window, tile count, record, class
// weights.  Returns its in-window voxel count (algorithmic pairs).
__device__ __forceinline__ int64_t prep_prim(const PrepArgs& A, int64_t gi) {
  const int f = (int)(gi / A.n_prims);
  const int i = (int)(gi - (int64_t)f * A.n_prims);
  const int C = A.n_classes;
  PrimRec rec;
  float* rw = reinterpret_cast<float*>(&rec);
#pragma unroll
  for (int k = 0; k < kRecWords; ++k) rw[k] = 0.0f;
  rec.lo[0] = rec.lo[1] = rec.lo[2] = 1;
  rec.hi[0] = rec.hi[1] = rec.hi[2] = 0;
  int count = 0;
  int64_t vol = 0;  // in-window voxels (algorithmic pairs) of this primitive
  float* lrow = A.lrows + gi * A.lrow;
  bool lrow_done = false;

  const bool valid_slot = !A.n_valid || i < A.n_valid[f];
  if (valid_slot) {
    const double* logits = A.logits + gi * C;
    PrimF64 P = prim_setup(A.mu + 3 * gi, A.scale + 3 * gi, A.rot + 4 * gi, A.opacity[gi],
                           A.eps + 2 * gi, logits, C);
    if (P.bad) {
      // first failing primitive wins: min over (index << 8 | bits)
      atomicMin(A.bad_word, ((unsigned long long)gi << 8) | (unsigned long long)P.bad);
    } else {
      // ---- window; identical expressions to the oracle ----
      double lo[3], hi[3], cc[3];
      const double res = A.grid.resolution;
      const double r = (double)A.cfg.neighborhood_radius +
                       ceil(__ddiv_rn(__dmul_rn(P.smax, A.cfg.window_extent), res));
      bool empty = false;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        cc[k] = floor(__ddiv_rn(__dsub_rn(P.mu[k], A.grid.origin[k]), res));
        if (A.cfg.truncate) {
          lo[k] = fmax(__dsub_rn(cc[k], r), 0.0);
          hi[k] = fmin(__dadd_rn(cc[k], r), (double)(A.grid.dims[k] - 1));
        } else {
          lo[k] = 0.0;
          hi[k] = (double)(A.grid.dims[k] - 1);
        }
        empty |= lo[k] > hi[k];
      }
      if (!empty && P.sigma > 0.0) {  // sigma = 0 primitives are skipped
        int ilo[3], ihi[3];
        vol = 1;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          ilo[k] = (int)lo[k];
          ihi[k] = (int)hi[k];
          rec.lo[k] = ilo[k];
          rec.hi[k] = ihi[k];
          vol *= (int64_t)(ihi[k] - ilo[k] + 1);
        }
        count = (ihi[0] / kTileX - ilo[0] / kTileX + 1) * (ihi[1] / kTileY - ilo[1] / kTileY + 1) *
                (ihi[2] / kTileZ - ilo[2] / kTileZ + 1);
        // ---- evaluation record ----
        // reference voxel: the centre voxel clamped into the window, so that
        // lattice offsets k = idx - cref stay small integers.
        double cref[3], d[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          cref[k] = fmin(fmax(cc[k], lo[k]), hi[k]);
          d[k] = (A.grid.origin[k] + (cref[k] + 0.5) * res) - P.mu[k];
        }
#pragma unroll
        for (int r2 = 0; r2 < 3; ++r2) {
          const double row[3] = {P.M[3 * r2] * res, P.M[3 * r2 + 1] * res, P.M[3 * r2 + 2] * res};
          const double g = P.M[3 * r2] * d[0] + P.M[3 * r2 + 1] * d[1] + P.M[3 * r2 + 2] * d[2];
          split_row(row, g, &rec.HL[3 * r2], &rec.G[r2]);
          rec.Ez[r2] = (float)row[2];
        }
        rec.a = (float)(2.0 / P.e2);
        rec.b = (float)(P.e2 / P.e1);
        rec.c = (float)(2.0 / P.e1);
        rec.cx = (float)cref[0];
        rec.cy = (float)cref[1];
        rec.cz = (float)cref[2];
        // class weights: logits (logit-sum) or softmax (prob-sum)
        double wmax = 1.0;  // max(1, sigma, max_k |class weight|)
        if (A.cfg.semantic_mode == 1) {
          double m = logits[0];
          for (int k = 1; k < C; ++k) m = fmax(m, logits[k]);
          double s = 0.0;
          for (int k = 0; k < C; ++k) s += exp(logits[k] - m);
          for (int k = 0; k < C; ++k) lrow[k] = (float)(exp(logits[k] - m) / s);
        } else {
          for (int k = 0; k < C; ++k) {
            lrow[k] = (float)logits[k];
            wmax = fmax(wmax, fabs(logits[k]));
          }
        }
        // Block-cull threshold of this primitive (sqv_common.cuh, kBlockCutMin):
        // cut = max(36, ln(N wmax / 2e-12)), so the primitive's dropped weights,
        // times its largest class weight, sum to < 2e-12 / N per voxel.
        // F >= max(|x'|)^(2/e1): the Chebyshev bound culls when max|x'| >
        // cut^(e1/2) (+0.1% margin, which dwarfs the exp2/log2 ulp error);
        // the block masks recover the field threshold as mcut^c >= cut.
        const double cut = fmax((double)kBlockCutMin,
                                log((double)A.n_prims * wmax) + kLnInvDropBound);
        rec.mcut = __double2float_ru(exp2(0.5 * P.e1 * log2(cut)) * 1.001);
        for (int k = C; k < A.lrow; ++k) lrow[k] = 0.0f;
        lrow[A.cm] = (float)P.sigma;
        // the padding column (never read as a class) carries wmax for the
        // block masks' per-tile cut (rounded up: the bound stays conservative)
        lrow[A.lrow - 1] = __double2float_ru(wmax);
        lrow_done = true;
      }
    }
  }
  if (!lrow_done)
    for (int k = 0; k < A.lrow; ++k) lrow[k] = 0.0f;
  reinterpret_cast<PrimRec*>(A.recs)[gi] = rec;
  A.counts[gi] = count;
  int* win = A.windows + 6 * gi;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    win[k] = rec.lo[k];
    win[3 + k] = rec.hi[k];
  }
  return vol;
}

__global__ void prep_kernel(PrepArgs A) {
  const int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t FN = (int64_t)A.n_frames * A.n_prims;
  unsigned long long v = gi < FN ? (unsigned long long)prep_prim(A, gi) : 0ull;
  // the entry total in 64 bits (counts[gi] was just written by this thread):
  // the int32 scan that follows wraps past 2^31 entries, so the host checks
  // this sum, not the scan's, before emit trusts the offsets
  unsigned long long e = gi < FN ? (unsigned long long)A.counts[gi] : 0ull;
  // one atomic per warp for each total (not one per primitive on a single
  // address)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v += __shfl_down_sync(0xffffffffu, v, o);
    e += __shfl_down_sync(0xffffffffu, e, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (v) atomicAdd(A.n_pairs, v);
    if (e) atomicAdd(A.n_entries, e);
  }
  // entries per frame (the per-frame binning's frame bases): one atomic per
  // frame segment of the warp (a warp spans at most a few frames)
  if (A.frame_count) {
    const int f = gi < FN ? (int)(gi / A.n_prims) : -1;
    const int c = gi < FN ? A.counts[gi] : 0;
    const unsigned peers = __match_any_sync(0xffffffffu, f);
    const int sum = __reduce_add_sync(peers, c);
    if (f >= 0 && sum && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&A.frame_count[f], sum);
  }
}

// K3: one thread per primitive; entries in (tz, ty, tx) order, primitive
// order preserved by the prefix offsets, so the stable radix sort by key
// yields ascending primitive ids per tile (the oracle's bins).
// K3: one warp per primitive writes its (tile key, primitive) entries —
// consecutive lanes to consecutive entries, so the stores coalesce — in
// tx-fastest order at the primitive's exclusive offset.  No atomics: tile
// offsets come from the sorted keys (tile_bounds_kernel).
__global__ void emit_kernel(EmitArgs A) {
  const int64_t FN = (int64_t)A.n_frames * A.n_prims;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t gi = w0; gi < FN; gi += nw) {
    const int cnt = A.counts[gi];
    if (cnt == 0) continue;
    const int f = (int)(gi / A.n_prims);
    const int i = (int)(gi - (int64_t)f * A.n_prims);
    const int* w = A.windows + 6 * gi;
    const int tx0 = w[0] / kTileX, ty0 = w[1] / kTileY, tz0 = w[2] / kTileZ;
    const int ntx = w[3] / kTileX - tx0 + 1, nty = w[4] / kTileY - ty0 + 1;
    const int64_t o = A.offs[gi];
    const uint32_t base = (uint32_t)f * (uint32_t)A.tiles_per_frame;
    for (int e = lane; e < cnt; e += 32) {
      const int dx = e % ntx, r = e / ntx, dy = r % nty, dz = r / nty;
      A.keys[o + e] = base + (uint32_t)(tx0 + dx + A.ntx * (ty0 + dy + A.nty * (tz0 + dz)));
      A.vals[o + e] = i;
    }
  }
}

// First sorted entry with key >= t (the upper levels of the search stay in
// L2/L1 for every thread).
__device__ __forceinline__ int64_t lower_bound_key(const uint32_t* keys, int64_t n, int64_t t) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)__ldg(keys + mid) < t)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// tile_off[t] = first sorted entry with key >= t (t = 0 .. n_tiles), one
// thread per tile.  With deep_min >= 0, tiles holding more than deep_min
// entries are also appended (unordered) to deep_tiles: the CUDA-core
// evaluator's complement walks that list instead of every tile.
__global__ void tile_bounds_kernel(const uint32_t* keys, int64_t n, int64_t n_tiles,
                                   int* tile_off, int deep_min, int* deep_tiles,
                                   int* deep_count) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t lo = lower_bound_key(keys, n, t < n_tiles ? t : n_tiles);
  if (t <= n_tiles) tile_off[t] = (int)lo;
  if (deep_min < 0) return;
  // the next tile's offset: the neighbour lane's, searched by the last lane
  int64_t nxt = __shfl_down_sync(0xffffffffu, lo, 1);
  if ((threadIdx.x & 31) == 31) nxt = lower_bound_key(keys, n, t + 1 < n_tiles ? t + 1 : n_tiles);
  if (t < n_tiles && nxt - lo > deep_min) deep_tiles[atomicAdd(deep_count, 1)] = (int)t;
}

}  // namespace sqv
