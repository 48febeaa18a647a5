// sqv_eval.cu — K5: per-tile evaluator with fused finalize (the hot kernel).
//
// One CTA owns one 8x8x16 voxel tile of one frame (SQV_TILE_*) and gathers
// the tile's primitive list (the bins, ascending primitive ids) in chunks
// staged in shared memory.  Each of the 8 warps owns a 4x4x8 voxel block,
// each lane a 1x1x4 z-column, so every (primitive, voxel) pair of the tile is
// evaluated by exactly one thread and every voxel accumulates its
// contributions in primitive order: the result is deterministic and does not
// depend on the batch or the GPU count.
//
// Per pair (core.py:237-282):
//   x' = local coordinates / scale  — hi/lo split lattice stepping (exact
//        offsets, no cancellation), see prep's split_row
//   F  = (|x'0|^a + |x'1|^a)^b + |x'2|^c          — 8 MUFU (lg2/ex2)
//   w  = exp(-F) (0 for F >= kFCut)               — 1 MUFU
//   v_o += sigma*w; v_c[k] += w*c_k               — C+1 FFMA, in registers
// Culling (never changes an output bit, see kFCut): a warp skips a primitive
// when its block misses the window, or when every live voxel has
// max|x'| > mcut, i.e. F > kFCut.
// Epilogue = finalize: free if v_o < tau, else the first
// argmax; dense grids and labels staged through shared memory and written
// as coalesced row segments (x-fastest layout).
#include "sqv_kernels.cuh"

namespace sqv {

namespace {

constexpr int kThreads = 256;
constexpr int kChunk = 64;  // primitives staged per chunk
constexpr int kVPT = 4;     // voxels per thread (consecutive z)

template <int CM>
struct EvalShape {
  static constexpr int kLRow = (CM + 1 + 3) & ~3;  // class weights + sigma, float4-padded
  static constexpr int kChunkBytes = kChunk * (kRecWords + kLRow) * 4;
};

template <int CM>
__global__ void __launch_bounds__(kThreads, 2) eval_kernel(EvalArgs A) {
  using S = EvalShape<CM>;
  extern __shared__ __align__(16) float smem[];
  float* s_rec = smem;                        // [kChunk][kRecWords]
  float* s_lw = smem + kChunk * kRecWords;    // [kChunk][kLRow]

  const int tile_g = blockIdx.x;
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
  const float xf = (float)x, yf = (float)y, z0f = (float)z0;

  float acc[kVPT][CM + 1];
#pragma unroll
  for (int v = 0; v < kVPT; ++v)
#pragma unroll
    for (int k = 0; k <= CM; ++k) acc[v][k] = 0.0f;

  const int beg = A.tile_off[tile_g], end = A.tile_off[tile_g + 1];
  const float* __restrict__ recs = A.recs;
  const float* __restrict__ lrows = A.lrows;
  const int64_t fbase = (int64_t)f * A.n_prims;

  for (int c0 = beg; c0 < end; c0 += kChunk) {
    const int n = min(kChunk, end - c0);
    __syncthreads();
    // stage records and class-weight rows of the chunk (L2-resident)
    for (int idx = tid; idx < n * (kRecWords / 4); idx += kThreads) {
      const int j = idx / (kRecWords / 4), q = idx - j * (kRecWords / 4);
      const int64_t g = fbase + A.prim_ids[c0 + j];
      reinterpret_cast<float4*>(s_rec)[idx] =
          __ldg(reinterpret_cast<const float4*>(recs + g * kRecWords) + q);
    }
    for (int idx = tid; idx < n * (S::kLRow / 4); idx += kThreads) {
      const int j = idx / (S::kLRow / 4), q = idx - j * (S::kLRow / 4);
      const int64_t g = fbase + A.prim_ids[c0 + j];
      reinterpret_cast<float4*>(s_lw)[idx] =
          __ldg(reinterpret_cast<const float4*>(lrows + g * A.lrow) + q);
    }
    __syncthreads();

    for (int j = 0; j < n; ++j) {
      const PrimRec& R = *reinterpret_cast<const PrimRec*>(s_rec + j * kRecWords);
      const int lox = R.lo[0], loy = R.lo[1], loz = R.lo[2];
      const int hix = R.hi[0], hiy = R.hi[1], hiz = R.hi[2];
      // warp-uniform: does this warp's 4x4x8 block meet the window?
      if (bx0 + 3 < lox || bx0 > hix || by0 + 3 < loy || by0 > hiy || bz0 + 7 < loz ||
          bz0 > hiz)
        continue;
      const bool in_xy = x >= lox && x <= hix && y >= loy && y <= hiy;
      const float fx = xf - R.cx, fy = yf - R.cy, fz = z0f - R.cz;
      // hi parts: exact; lo parts: small
      float h0 = fmaf(fz, R.H[2], fmaf(fy, R.H[1], fx * R.H[0]));
      float h1 = fmaf(fz, R.H[5], fmaf(fy, R.H[4], fx * R.H[3]));
      float h2 = fmaf(fz, R.H[8], fmaf(fy, R.H[7], fx * R.H[6]));
      float l0 = fmaf(fz, R.L[2], fmaf(fy, R.L[1], fmaf(fx, R.L[0], R.G[0])));
      float l1 = fmaf(fz, R.L[5], fmaf(fy, R.L[4], fmaf(fx, R.L[3], R.G[1])));
      float l2 = fmaf(fz, R.L[8], fmaf(fy, R.L[7], fmaf(fx, R.L[6], R.G[2])));
      const float mcut = R.mcut;
      float p0[kVPT], p1[kVPT], p2[kVPT];
      bool live[kVPT];
      bool any = false;
#pragma unroll
      for (int v = 0; v < kVPT; ++v) {
        p0[v] = h0 + l0;
        p1[v] = h1 + l1;
        p2[v] = h2 + l2;
        h0 += R.H[2];
        h1 += R.H[5];
        h2 += R.H[8];
        l0 += R.L[2];
        l1 += R.L[5];
        l2 += R.L[8];
        const int z = z0 + v;
        const float m = fmaxf(fmaxf(fabsf(p0[v]), fabsf(p1[v])), fabsf(p2[v]));
        live[v] = in_xy && z >= loz && z <= hiz && m <= mcut;
        any |= live[v];
      }
      if (!__any_sync(0xffffffffu, any)) continue;
      const float a = R.a, b = R.b, c = R.c;
      float w[kVPT];
#pragma unroll
      for (int v = 0; v < kVPT; ++v) {
        const float F = field_F(p0[v], p1[v], p2[v], a, b, c);
        w[v] = (live[v] && F < kFCut) ? ex2(-F * kLog2e) : 0.0f;
      }
      const float* lw = s_lw + j * S::kLRow;
#pragma unroll
      for (int k = 0; k <= CM; ++k) {
        const float ck = lw[k];
#pragma unroll
        for (int v = 0; v < kVPT; ++v) acc[v][k] = fmaf(w[v], ck, acc[v][k]);
      }
    }
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
    for (int row = warp; row < 64; row += kThreads / 32) {
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
}

template <int CM>
int launch_cm(const EvalArgs& A, int n_tiles, cudaStream_t s) {
  using S = EvalShape<CM>;
  const int stage_bytes = 512 * (CM * 4 + 4 + 1);
  const int smem = S::kChunkBytes > stage_bytes ? S::kChunkBytes : stage_bytes;
  if (cudaFuncSetAttribute(eval_kernel<CM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
      cudaSuccess)
    return check_launch("eval_kernel attribute");
  eval_kernel<CM><<<n_tiles, kThreads, smem, s>>>(A);
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
  switch (cm) {
    case 2: return launch_cm<2>(A, n_tiles, s);
    case 4: return launch_cm<4>(A, n_tiles, s);
    case 8: return launch_cm<8>(A, n_tiles, s);
    case 12: return launch_cm<12>(A, n_tiles, s);
    case 16: return launch_cm<16>(A, n_tiles, s);
    case 18: return launch_cm<18>(A, n_tiles, s);
    case 24: return launch_cm<24>(A, n_tiles, s);
    case 32: return launch_cm<32>(A, n_tiles, s);
    default: return set_error(SQV_ERR_UNSUPPORTED, "no evaluator for %d classes", cm);
  }
}

}  // namespace sqv
