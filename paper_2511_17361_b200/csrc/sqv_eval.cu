// sqv_eval.cu — K5: per-tile evaluator with fused finalize (the hot kernel).
//
// One CTA owns one 8x8x16 voxel tile of one frame (SQV_TILE_*) and gathers
// the tile's primitive list (the bins, ascending primitive ids), staged in
// shared memory in chunks of up to kChunk primitives (one chunk for almost
// every tile).  Each of the 8 warps owns a 4x4x8 voxel block, each lane a
// 1x1x4 z-column, so every (primitive, voxel) pair of the tile is evaluated by
// exactly one thread and every voxel accumulates its contributions in
// primitive order: the result is deterministic and does not depend on the
// batch or the GPU count.
//
// Per chunk each warp first builds a bitmask of the staged primitives whose
// window meets its block (lane-parallel test + ballot), then walks only the
// set bits, so a primitive that misses a warp costs that warp nothing.
//
// Per pair (core.py:237-282):
//   x' = local coordinates / scale  — hi/lo split lattice stepping (exact
//        offsets, no cancellation), see prep's split_row
//   F  = (|x'0|^a + |x'1|^a)^b + |x'2|^c          — 7 MUFU (field_F7)
//   w  = exp(-F) (0 for F >= kFCut)               — 1 MUFU
//   v_o += sigma*w; v_c[k] += w*c_k               — C+1 FFMA, in registers
// Culling (block_may_hit): skipped when F exceeds the primitive's block-cull
// threshold on every voxel of the warp's block (every dropped weight is below
// exp(-cut); see kBlockCutMin in sqv_common.cuh).
// Epilogue = finalize: free if v_o < tau, else the first
// argmax; dense grids and labels staged through shared memory and written
// as coalesced row segments (x-fastest layout).
#include "sqv_kernels.cuh"
#include "sqv_pair.cuh"

namespace sqv {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kChunk = 256;            // primitives staged per chunk
constexpr int kMaskWords = kChunk / 32;

template <int CM>
struct EvalShape {
  static constexpr int kLRow = (CM + 1 + 3) & ~3;  // class weights + sigma, float4-padded
  static constexpr int kChunkBytes = kChunk * (kRecWords + kLRow) * 4 + kWarps * kMaskWords * 4;
  static constexpr int kStageBytes = 512 * (CM * 4 + 4 + 1);
  static constexpr int kSmem = kChunkBytes > kStageBytes ? kChunkBytes : kStageBytes;
};

template <int CM, int FIELD>
__global__ void __launch_bounds__(kThreads, (CM <= 18 ? 2 : 1)) eval_kernel(EvalArgs A) {
  using S = EvalShape<CM>;
  extern __shared__ __align__(16) float smem[];
  float* s_rec = smem;                                   // [kChunk][kRecWords]
  float* s_lw = smem + kChunk * kRecWords;               // [kChunk][kLRow]
  unsigned* s_mask = reinterpret_cast<unsigned*>(s_lw + kChunk * S::kLRow);  // [kWarps][kMaskWords]

  // One tile per CTA, or — as the deep-tile complement of the tensor-core
  // evaluator — a grid-stride walk over the tiles with more than
  // ffma_min_entries entries, listed by tile_bounds_kernel (the others are
  // the tensor-core kernel's).
  const bool listed = A.ffma_min_entries >= 0;
  const int n_walk = listed ? *A.deep_count : A.n_tiles;
  for (int it = blockIdx.x; it < n_walk; it += gridDim.x) {
  const int tile_g = listed ? A.deep_tiles[it] : it;
  const int f = tile_g / A.tiles_per_frame;
  const int t = tile_g - f * A.tiles_per_frame;
  const int tx = t % A.ntx;
  const int ty = (t / A.ntx) % A.nty;
  const int tz = t / (A.ntx * A.nty);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // warp block (4x4x8) and lane column (1x1x4)
  const int bx0 = tx * kTileX + (warp & 1) * 4;
  const int by0 = ty * kTileY + ((warp >> 1) & 1) * 4;
  const int bz0 = tz * kTileZ + (warp >> 2) * 8;
  const int x = bx0 + (lane & 3);
  const int y = by0 + ((lane >> 2) & 3);
  const int z0 = bz0 + (lane >> 4) * 4;

  float acc[kVPT][CM + 1];
#pragma unroll
  for (int v = 0; v < kVPT; ++v)
#pragma unroll
    for (int k = 0; k <= CM; ++k) acc[v][k] = 0.0f;

  const int beg = A.tile_off[tile_g], end = A.tile_off[tile_g + 1];
  const int64_t fbase = (int64_t)f * A.n_prims;

  for (int c0 = beg; c0 < end; c0 += kChunk) {
    const int n = min(kChunk, end - c0);
    __syncthreads();
    // stage records and class-weight rows of the chunk (L2-resident)
    for (int idx = tid; idx < n * (kRecWords / 4); idx += kThreads) {
      const int j = idx / (kRecWords / 4), q = idx - j * (kRecWords / 4);
      const int64_t g = fbase + A.prim_ids[c0 + j];
      reinterpret_cast<float4*>(s_rec)[idx] =
          __ldg(reinterpret_cast<const float4*>(A.recs + g * kRecWords) + q);
    }
    for (int idx = tid; idx < n * (S::kLRow / 4); idx += kThreads) {
      const int j = idx / (S::kLRow / 4), q = idx - j * (S::kLRow / 4);
      const int64_t g = fbase + A.prim_ids[c0 + j];
      reinterpret_cast<float4*>(s_lw)[idx] =
          __ldg(reinterpret_cast<const float4*>(A.lrows + g * A.lrow) + q);
    }
    __syncthreads();
    // per-warp hit masks: which staged primitives' windows meet this block
    for (int q = 0; q * 32 < n; ++q) {
      const int j = q * 32 + lane;
      bool hit = false;
      if (j < n) {
        hit = block_may_hit(*reinterpret_cast<const PrimRec*>(s_rec + j * kRecWords), bx0, by0,
                            bz0);
      }
      const unsigned m = __ballot_sync(0xffffffffu, hit);
      if (lane == 0) s_mask[warp * kMaskWords + q] = m;
    }
    __syncwarp();

    unsigned long long st_mufu = 0, st_blocks = 0;  // instrumentation (A.stats)
    for (int q = 0; q * 32 < n; ++q) {
      unsigned m = s_mask[warp * kMaskWords + q];
      while (m) {
        const int j = q * 32 + __ffs(m) - 1;
        m &= m - 1;
        const PrimRec& R = *reinterpret_cast<const PrimRec*>(s_rec + j * kRecWords);
        st_mufu += mufu_per_block(FIELD, wants_acc<FIELD>(R));
        ++st_blocks;
        float w[kVPT];
        pair_weights<FIELD>(R, x, y, z0, w);
        const float4* lw = reinterpret_cast<const float4*>(s_lw + j * S::kLRow);
#pragma unroll
        for (int k4 = 0; k4 < S::kLRow / 4; ++k4) {
          const float4 c4 = lw[k4];
          const float cc[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int k = 4 * k4 + e;
            if (k <= CM) {
#pragma unroll
              for (int v = 0; v < kVPT; ++v) acc[v][k] = fmaf(w[v], cc[e], acc[v][k]);
            }
          }
        }
      }
    }
    if (lane == 0) add_stats(A.stats, st_mufu, st_blocks);
  }

  // ---- epilogue: finalize + staged coalesced stores ----------------------
  const int C = A.n_classes;
  uint8_t lab[kVPT];
#pragma unroll
  for (int v = 0; v < kVPT; ++v) {
    const float vo = acc[v][CM];
    int best = 0;
    float bv = acc[v][0];
#pragma unroll
    for (int k = 1; k < CM; ++k)
      if (k < C && acc[v][k] > bv) {
        bv = acc[v][k];
        best = k;
      }
    lab[v] = (vo < A.tau) ? (uint8_t)A.free_label : (uint8_t)best;
  }
  const int nx = A.nx, ny = A.ny, nz = A.nz;
  const int x_t = tx * kTileX, y_t = ty * kTileY;
  const int64_t V = (int64_t)nx * ny * nz;
  // stage one z-half (8 layers = 512 voxels) at a time
  float* s_vc = smem;                 // [512][C]
  float* s_vo = smem + 512 * C;       // [512]
  uint8_t* s_lab = reinterpret_cast<uint8_t*>(s_vo + 512);
  for (int half = 0; half < 2; ++half) {
    const int zh = tz * kTileZ + half * 8;
    if (zh >= nz) break;  // uniform
    __syncthreads();
    if ((warp >> 2) == half) {
#pragma unroll
      for (int v = 0; v < kVPT; ++v) {
        const int zl = (z0 + v) - zh;  // 0..7
        const int loc = (x - x_t) + kTileX * ((y - y_t) + kTileY * zl);
        if (A.v_c) {
#pragma unroll
          for (int k = 0; k < CM; ++k)
            if (k < C) s_vc[loc * C + k] = acc[v][k];
        }
        s_vo[loc] = acc[v][CM];
        s_lab[loc] = lab[v];
      }
    }
    __syncthreads();
    const int xw = min(kTileX, nx - x_t);  // valid voxels per row
    // 64 rows (8 z x 8 y) of 8 voxels
    for (int row = warp; row < 64; row += kWarps) {
      const int yl = row & 7, zl = row >> 3;
      const int yy = y_t + yl, zz = zh + zl;
      if (yy >= ny || zz >= nz) continue;
      const int64_t gv = (int64_t)f * V + (int64_t)x_t + (int64_t)nx * (yy + (int64_t)ny * zz);
      if (A.v_c) {
        const int nel = xw * C;
        const float* src = s_vc + row * kTileX * C;
        float* dst = A.v_c + gv * C;
        for (int e = lane; e < nel; e += 32) dst[e] = src[e];
      }
      if (lane < xw) {
        if (A.v_o) A.v_o[gv + lane] = s_vo[row * kTileX + lane];
        A.labels[gv + lane] = s_lab[row * kTileX + lane];
      }
    }
  }
  }  // tile loop
}

template <int CM>
int launch_cm(const EvalArgs& A, int n_tiles, int field, cudaStream_t s) {
  using S = EvalShape<CM>;
  auto kern = field == 9 ? eval_kernel<CM, 9> : field == 8 ? eval_kernel<CM, 8> : field == 6 ? eval_kernel<CM, 6> : eval_kernel<CM, 7>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::kSmem) !=
      cudaSuccess)
    return check_launch("eval_kernel attribute");
  int grid = n_tiles;
  if (A.ffma_min_entries >= 0) {  // deep tiles only: a grid-stride walk
    static int n_sm = 0;
    if (!n_sm) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
      if (n_sm < 1) n_sm = 148;
    }
    grid = n_tiles < 2 * n_sm ? n_tiles : 2 * n_sm;
  }
  kern<<<grid, kThreads, S::kSmem, s>>>(A);
  count_launch();
  return check_launch("eval_kernel");
}

}  // namespace

int eval_cm_for(int C) {
  if (C <= 0) return 0;
  if (C <= 2) return 2;
  if (C <= 4) return 4;
  if (C <= 8) return 8;
  if (C <= 12) return 12;
  if (C <= 16) return 16;
  if (C <= 18) return 18;
  if (C <= 24) return 24;
  if (C <= 32) return 32;
  return 0;
}

int eval_launch(const EvalArgs& A, int cm, int n_tiles, cudaStream_t s) {
  if (n_tiles <= 0) return SQV_OK;
  const int field = (A.field == 9 || A.field == 8 || A.field == 6) ? A.field : 7;
  switch (cm) {
    case 2: return launch_cm<2>(A, n_tiles, field, s);
    case 4: return launch_cm<4>(A, n_tiles, field, s);
    case 8: return launch_cm<8>(A, n_tiles, field, s);
    case 12: return launch_cm<12>(A, n_tiles, field, s);
    case 16: return launch_cm<16>(A, n_tiles, field, s);
    case 18: return launch_cm<18>(A, n_tiles, field, s);
    case 24: return launch_cm<24>(A, n_tiles, field, s);
    case 32: return launch_cm<32>(A, n_tiles, field, s);
    default: return set_error(SQV_ERR_UNSUPPORTED, "no evaluator for %d classes", cm);
  }
}

}  // namespace sqv
