// sqv_kernels.cuh — kernel argument blocks and host-side launchers.
#pragma once

#include "sqv_common.cuh"

namespace sqv {

struct PrepArgs {
  const double *mu, *scale, *rot, *opacity, *eps, *logits;
  const int32_t* n_valid;
  int n_frames, n_prims, n_classes;
  int cm;    // padded class count of the evaluator instantiation (sigma at lrow[cm])
  int lrow;  // floats per class-weight row
  sqv_grid grid;
  sqv_cfg cfg;
  float* recs;   // [FN][kRecWords]
  float* lrows;  // [FN][lrow]
  int* counts;   // [FN] tiles overlapped
  int* windows;  // [FN][6]
  unsigned long long* bad_word;
  unsigned long long* n_pairs;
  // 64-bit sum of counts[]: the (tile, primitive) entry total, checked on the
  // host before the 32-bit scan offsets and emit are trusted
  unsigned long long* n_entries;
  int* frame_count;  // [F] entries per frame (per-frame binning), or NULL
};

// per-frame binning (sqv_bin.cu): tile lists, offsets, deep list, masks
struct BinArgs {
  int n_frames, n_prims;
  int tiles_per_frame, ntx, nty;
  const int* counts;       // [FN] tiles per primitive (prep)
  const int* windows;      // [FN][6] clipped voxel windows (prep)
  const int* frame_count;  // [F] entries per frame (prep)
  uint32_t* keys;          // [E] global tile id per entry
  int* vals;               // [E] frame-local primitive id per entry
  int* tile_off;           // [F*T + 1]
  int deep_min;            // tiles with more entries go to deep_tiles (-1: none)
  int* deep_tiles;
  int* deep_count;
  const float* recs;       // block masks (bmask NULL: none)
  const float* lrows;
  int lrow;
  float acc_c;
  uint32_t* bmask;
};
size_t bin_frames_smem(int tiles_per_frame);
bool bin_frames_supported(int tiles_per_frame);
int bin_frames_launch(const BinArgs& A, cudaStream_t s);

struct EmitArgs {
  int n_frames, n_prims;
  int tiles_per_frame, ntx, nty;
  const int* counts;
  const int* offs;
  const int* windows;
  uint32_t* keys;
  int* vals;
};

struct EvalArgs {
  const float* recs;
  const float* lrows;
  const int* tile_off;
  const int* prim_ids;
  int n_prims, n_classes, lrow;
  int tiles_per_frame, ntx, nty;
  int nx, ny, nz;
  float tau;
  int free_label;
  int field;  // 7 (default) or 9: field_F7 / field_F (A/B diagnostics, env SQV_FIELD)
  uint8_t* labels;
  float* v_o;
  float* v_c;
  int n_tiles;        // F * tiles per frame
  // accumulation-depth split: the tensor-core evaluator takes tiles with at
  // most tc_max_entries (tile, primitive) entries, the CUDA-core one those
  // with more than ffma_min_entries (-1: all tiles), listed by tile_bounds_kernel
  int tc_max_entries;
  int ffma_min_entries;
  const int* deep_tiles;  // tiles with more than ffma_min_entries entries (unordered)
  const int* deep_count;  // their number (device)
  int* tile_counter;  // zeroed device int: the persistent evaluator's work counter
  int64_t n_entries;  // (tile, primitive) entries of the batch
  // optional instrumentation (sqv_stats_attach): [0] += MUFU ops issued by
  // the evaluators (thread level), [1] += evaluated (primitive, voxel) pairs
  // (warp blocks run x 128, window-dead voxels of partial blocks included)
  unsigned long long* stats;
  // per entry: bit b = may hit warp block b, bit 8+b = covers it, bit 16 =
  // strict mode's accurate-log primitive (c > SQV_ACC_C)
  const uint32_t* bmask;
};

// per (tile, primitive) entry: the 8 warp-block tests of the tensor-core
// evaluator (block_may_hit / block_inside), computed once, in parallel
int block_masks_launch(const uint32_t* sorted_keys, const int* sorted_ids, int64_t n_entries,
                       const float* recs, const float* lrows, int lrow, const int* tile_off,
                       int tiles_per_frame, int ntx, int nty, int n_prims, float acc_c,
                       uint32_t* bmask, cudaStream_t s);

__global__ void prep_kernel(PrepArgs A);
__global__ void emit_kernel(EmitArgs A);
__global__ void tile_bounds_kernel(const uint32_t* keys, int64_t n, int64_t n_tiles,
                                   int* tile_off, int deep_min, int* deep_tiles,
                                   int* deep_count);

// exclusive scan of n int32 values; out has n+1 entries (out[n] = total);
// if total64 != nullptr the total is also stored there.  tmp needs
// scan_tmp_ints(n) ints.  The running sums are int32: callers bound the
// total below 2^31 first (sqv_voxelize checks prep's 64-bit entry total).
int64_t scan_tmp_ints(int64_t n);
int scan_exclusive(const int* in, int* out, int64_t n, int* tmp, long long* total64,
                   cudaStream_t s);

// stable LSD radix sort of (keys, vals) by the low `bits` bits of key.
// Result lands in (keys, vals) or (keys_alt, vals_alt); returns 0 or 1 in *which.
int64_t radix_tmp_ints(int64_t n);
int radix_sort(uint32_t* keys, int* vals, uint32_t* keys_alt, int* vals_alt, int64_t n, int bits,
               int* tmp, int* which, cudaStream_t s);

// MUFU ops per evaluated voxel of each field form, times 128 voxels per warp
// block: strict 7 (3 lg2 + 4 ex2), strict accurate-log 4 (ex2 only), fast 6.5
// (one voxel pair's t on the FMA pipe), the 8- and 9-MUFU diagnostic forms
__host__ __device__ constexpr unsigned long long mufu_per_block(int field, bool acc) {
  return field == 6 ? (acc ? 512ull : 896ull)
                    : field == 7 ? 832ull : field == 8 ? 1024ull : 1152ull;
}
__device__ __forceinline__ void add_stats(unsigned long long* st, unsigned long long mufu,
                                          unsigned long long blocks) {
  if (st) {
    atomicAdd(st, mufu);
    atomicAdd(st + 1, blocks * 128ull);
  }
}

// evaluator
int eval_cm_for(int C);  // padded class count for C (0 if unsupported)
int eval_launch(const EvalArgs& A, int cm, int n_tiles_total, cudaStream_t s);
// tensor-core (tcgen05) evaluator, CM <= 24
bool eval_tc_supported(int cm);
int eval_tc_launch(const EvalArgs& A, int cm, int n_tiles_total, cudaStream_t s);

// misc kernels
int finalize_launch(const float* v_o, const float* v_c, int64_t n, int C, float tau, int free_label,
                    uint8_t* labels, cudaStream_t s);
int confusion_launch(const uint8_t* pred, const uint8_t* gt, int64_t n, int C, int64_t* cm,
                     cudaStream_t s);
int microbench(int which, double* ops_per_s, cudaStream_t s);
// device scene generation (sqv_gen.cu)
struct GenArgs {
  uint64_t seed;
  int64_t first_frame;
  int n_frames, n_prims, n_classes;
  double lo[3], hi[3];
  double smin, smax, emin;
  double *mu, *scale, *rot, *opacity, *eps, *logits;
};
int gen_launch(const GenArgs& A, cudaStream_t s);

// ray_iou (sqv_ray.cu)
constexpr int kMaxRayThr = 16;
struct RayArgs {
  const uint8_t* pred;
  const uint8_t* gt;
  int dims[3];
  double org[3];
  double res;
  int n_classes;
  int n_frames;
  int64_t n_rays;
  const double* origins;
  const double* dirs;
  int n_thr;
  double thr[kMaxRayThr];
  unsigned long long* counts;
  double* d_pred;
  int32_t* c_pred;
  double* d_gt;
  int32_t* c_gt;
};
int ray_iou_launch(const RayArgs& A, cudaStream_t s);

int density_launch(const sqv_prims* P, const double* points, const int32_t* pair_prim,
                   int64_t n, float* F, float* density, cudaStream_t s);

}  // namespace sqv
