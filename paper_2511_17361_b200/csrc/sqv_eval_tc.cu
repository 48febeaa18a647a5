// sqv_eval_tc.cu — K5 on the 5th-generation tensor cores (tcgen05 + TMEM).
//
// Same tile/warp/lane decomposition and the same per-pair weights as the
// FFMA evaluator (sqv_pair.cuh), but the accumulation
//
//     [v_c | v_o](voxel, :) += w(voxel, prim) * [c_prim | sigma_prim]
//
// is what it is — a GEMM, W[128 voxels x K prims] * L[K prims x 32] per warp —
// so it runs as tcgen05.mma.kind::tf32 with the accumulator in TMEM:
//
//   * each warp owns one M=128 block (its 4x4x8 voxels: row = lane*4 + v);
//   * for every primitive its 128 weights go to the warp's A operand in shared
//     memory and the primitive's class weights + sigma to the warp's B operand
//     (N = 32), both MN-major in the 128B_BASE32B swizzle (the MN-major mode
//     tf32 supports): one conflict-free STS.128 per lane for A (row =
//     lane*4 + voxel slot), one STS.32 per lane for B;
//   * every K = 8 primitives one elected lane issues three MMAs — W_hi*L_hi,
//     W_hi*L_lo, W_lo*L_hi (3xTF32 split: hi = top 11 bits, lo = remainder) —
//     and commits them to the warp's mbarrier; the A/B buffers are reused once
//     that barrier flips;
//   * D (128 x 32 fp32) lives in TMEM columns [32*warp, 32*warp + 32).
//
// The split products carry ~2^-21 relative error per term (vs 2^-24 for FFMA)
// — two orders below the 1e-5 density tolerance — and every voxel still sums
// its primitives in ascending order within each K step, so results are
// deterministic.  Epilogue: tcgen05.ld (warp w reads TMEM lanes 32*(w%4)..+31)
// -> finalize (tau, first argmax) -> staged coalesced stores.
#include "sqv_eval_tc_impl.cuh"

namespace sqv {

// launch_tc<CM> is instantiated in sqv_eval_tc_cm*.cu
extern template int launch_tc<2>(const EvalArgs&, int, int, cudaStream_t);
extern template int launch_tc<4>(const EvalArgs&, int, int, cudaStream_t);
extern template int launch_tc<8>(const EvalArgs&, int, int, cudaStream_t);
extern template int launch_tc<12>(const EvalArgs&, int, int, cudaStream_t);
extern template int launch_tc<16>(const EvalArgs&, int, int, cudaStream_t);
extern template int launch_tc<18>(const EvalArgs&, int, int, cudaStream_t);
extern template int launch_tc<24>(const EvalArgs&, int, int, cudaStream_t);

namespace {

// Per (tile, primitive) entry: which of the tile's 8 warp blocks the
// primitive may reach (bits 0-7) and which blocks lie entirely inside its
// window (bits 8-15).  The cull decisions are those of block_may_hit (window
// overlap, the Chebyshev box bound, the nearest-corner field bound, all
// conservative); the shared parts are computed once per entry (local block
// centres differ by fixed lattice steps), and a block whose nearest local
// corner is deep inside — (2^b + 1) max|x'|^c well below the primitive's cut
// — is marked without the 8-MUFU field test.  Bit 16 flags strict mode's
// accurate-log primitives (c > acc_c), so the evaluator's list build needs
// only the mask.  A "hit" that could have been
// culled only costs evaluation work: those pairs get their exact FP32 w.
__global__ void block_masks_kernel(const uint32_t* keys, const int* ids, int64_t n,
                                   const float* recs, const float* lrows, int lrow,
                                   const int* tile_off, int tiles_per_frame, int ntx, int nty,
                                   int n_prims, float acc_c, uint32_t* bmask) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const uint32_t key = keys[e];
  const int f = (int)(key / (uint32_t)tiles_per_frame);
  const int t = (int)(key - (uint32_t)f * (uint32_t)tiles_per_frame);
  const int tx = t % ntx, ty = (t / ntx) % nty, tz = t / (ntx * nty);
  PrimRec R;
  const float4* src = reinterpret_cast<const float4*>(recs + ((int64_t)f * n_prims + ids[e]) *
                                                             kRecWords);
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
  const float wmax = __ldg(lrows + ((int64_t)f * n_prims + ids[e]) * lrow + (lrow - 1));
  const int e_tile = __ldg(tile_off + key + 1) - __ldg(tile_off + key);
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
  for (int bb = 0; bb < kWarps; ++bb) {
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
  bmask[e] = m;
}

}  // namespace

bool eval_tc_supported(int cm) { return cm <= 24; }

int block_masks_launch(const uint32_t* sorted_keys, const int* sorted_ids, int64_t n_entries,
                       const float* recs, const float* lrows, int lrow, const int* tile_off,
                       int tiles_per_frame, int ntx, int nty, int n_prims, float acc_c,
                       uint32_t* bmask, cudaStream_t s) {
  if (n_entries <= 0) return SQV_OK;
  block_masks_kernel<<<(unsigned)((n_entries + 127) / 128), 128, 0, s>>>(
      sorted_keys, sorted_ids, n_entries, recs, lrows, lrow, tile_off, tiles_per_frame, ntx, nty,
      n_prims, acc_c, bmask);
  count_launch();
  return check_launch("block_masks_kernel");
}

int eval_tc_launch(const EvalArgs& A, int cm, int n_tiles, cudaStream_t s) {
  if (n_tiles <= 0) return SQV_OK;
  const int field = (A.field == 9 || A.field == 8 || A.field == 6) ? A.field : 7;
  switch (cm) {
    case 2: return launch_tc<2>(A, n_tiles, field, s);
    case 4: return launch_tc<4>(A, n_tiles, field, s);
    case 8: return launch_tc<8>(A, n_tiles, field, s);
    case 12: return launch_tc<12>(A, n_tiles, field, s);
    case 16: return launch_tc<16>(A, n_tiles, field, s);
    case 18: return launch_tc<18>(A, n_tiles, field, s);
    case 24: return launch_tc<24>(A, n_tiles, field, s);
    default: return set_error(SQV_ERR_UNSUPPORTED, "no tensor-core evaluator for %d classes", cm);
  }
}

}  // namespace sqv
