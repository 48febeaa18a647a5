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

// Per (tile, primitive) entry of the radix-sorted bins: its block mask
// (sqv_pair.cuh entry_block_mask: bits 0-7 may hit warp block b, 8-15 block
// wholly inside the window, 16 strict mode's accurate-log primitive).  The
// per-frame binning (sqv_bin.cu) computes the same masks inside its kernel.
__global__ void block_masks_kernel(const uint32_t* keys, const int* ids, int64_t n,
                                   const float* recs, const float* lrows, int lrow,
                                   const int* tile_off, int tiles_per_frame, int ntx, int nty,
                                   int n_prims, float acc_c, uint32_t* bmask) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const uint32_t key = keys[e];
  const int f = (int)(key / (uint32_t)tiles_per_frame);
  const int t = (int)(key - (uint32_t)f * (uint32_t)tiles_per_frame);
  const int64_t g = (int64_t)f * n_prims + ids[e];
  const int e_tile = __ldg(tile_off + key + 1) - __ldg(tile_off + key);
  bmask[e] = entry_block_mask(recs + g * kRecWords, __ldg(lrows + g * lrow + (lrow - 1)), e_tile,
                              t % ntx, (t / ntx) % nty, t / (ntx * nty), acc_c);
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
