// sqv_eval_tc_impl.cuh — the tcgen05 evaluator kernel template (K5) and its
// per-class-count launcher, shared by the translation units that
// instantiate them (sqv_eval_tc_cm*.cu; split so the build compiles them
// in parallel).  Design notes: the header comment of sqv_eval_tc.cu.
#pragma once

#include "sqv_kernels.cuh"
#include "sqv_pair.cuh"
#include "sqv_tc.cuh"

#include <cstdlib>
#include <type_traits>

namespace sqv {

namespace {

constexpr int kThreads = 256;
constexpr int kPersistentBelow = 64;  // mean primitives per tile
constexpr int kWarps = 8;
constexpr int kK = 8;        // K per tcgen05.mma.kind::tf32
constexpr int kN = 32;       // class weights + sigma, padded
constexpr int kTmemCols = kWarps * kN;  // 256 -> two CTAs per SM fill the 512 columns
constexpr uint32_t kIdesc = tc::idesc_tf32(128, kN, 1, 1);

template <int CM, int NW = 8>
struct TcShape {
  static_assert(CM + 1 <= kN, "sigma column must fit in N");
  static_assert(NW == 8 || NW == 4, "8 or 4 warp blocks per CTA");
  static constexpr int kLRow = (CM + 1 + 3) & ~3;
#ifdef SQV_CHUNK
  static constexpr int kChunk8 = CM <= 18 ? SQV_CHUNK : 104;
#else
  static constexpr int kChunk8 = CM <= 18 ? 120 : 104;
#endif
  // 4-warp CTAs (four per SM; one z half of a bin tile) stage at most
  // 2 x 128 threads / 2 = 64 primitives per chunk and fit 4 x 55 KB of shared
  // memory with 48.  (Measured for sparse batches, config 1: fast +6.4%,
  // strict -0.6% against 8 warps; not instantiated.)
  static constexpr int kChunk = NW == 8 ? kChunk8 : (CM <= 18 ? 48 : 40);
  // operand buffers (1 KB aligned): per warp A_hi, A_lo (4 KB each), B_hi, B_lo (1 KB each)
  static constexpr int kA = 0;
  static constexpr int kB = kA + NW * 2 * 4096;
  // staged primitives: record (40 words) + class weights/sigma (kLRow) each
  static constexpr int kStride = kRecWords + kLRow;  // words
  static constexpr int kRec = kB + NW * 2 * 1024;
  // per-warp hit lists (offsets of staged primitives in 16 B units): primitives
  // whose window covers the warp's whole block from the front, the rest from
  // the back
  static constexpr int kList = kRec + kChunk * kStride * 4;
  static_assert(kStride % 4 == 0, "16-byte aligned staging");
  static constexpr int kBm = kList + NW * kChunk * 2;  // staged block masks (u16)
  static constexpr int kAcc = kBm + kChunk * 2;  // strict: per-warp u8 lists of accurate-log primitives
  static constexpr int kBar = (kAcc + NW * kChunk + 7) & ~7;
  static constexpr int kMisc = kBar + NW * 8;   // tmem base (4 B) + has flags (NW x 4 B)
  static constexpr int kEnd = kMisc + 4 + NW * 4 + 4;  // + next-tile slot
  // epilogue staging (aliases kA..): z layers padded by 8 words so the 4 lanes
  // holding z-adjacent voxels hit different banks
  static constexpr int kStage = 2 * NW * ((64 * CM + 8) * 4 + 72 * 4 + 72);
  static constexpr int kBody = kEnd > kStage ? kEnd : kStage;
  static constexpr int kSmem = kBody + 1024;               // + alignment slack
  static_assert((16 / NW) * (kSmem + 1024) <= 228 * 1024, "CTAs per SM by shared memory");
  static_assert(kStage <= kMisc, "staging must not overwrite the flags");
};

__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

// Epilogue of one tile (all NW warps of the CTA; every MMA of the tile
// complete, published by a CTA barrier): TMEM -> finalize (tau, first argmax,
// SPEC.md:365-369) -> shared-memory staging (aliases the operand buffers) ->
// coalesced row stores.  NW = 8: the whole 8x8x16 tile (16 z layers); NW = 4:
// one z half of it (8 layers starting at z offset zh), warp blocks 0..3.
template <int CM, int NW = 8>
__device__ __forceinline__ void tile_epilogue(const EvalArgs& A, uint8_t* smem, const int* s_has,
                                              uint32_t tmem_base, int warp, int lane, int f,
                                              int tx, int ty, int tz, int zh = 0) {
  static_assert(NW == 8 || NW == 4, "8 or 4 warp blocks per CTA");
  constexpr int LZ = 2 * NW;          // z layers of the CTA's voxels
  constexpr int RPW = 8 / NW;         // y rows per warp in the store phase
  const int C = A.n_classes;
  const int nx = A.nx, ny = A.ny, nz = A.nz;
  const int x_t = tx * kTileX, y_t = ty * kTileY, z_t = tz * kTileZ + zh;
  const int zpc = 64 * C + 8;                          // padded z pitches
  constexpr int zpo = 72;
  float* s_vc = reinterpret_cast<float*>(smem);        // [LZ][zpc]
  float* s_vo = s_vc + LZ * zpc;                       // [LZ][zpo]
  uint8_t* s_lab = reinterpret_cast<uint8_t*>(s_vo + LZ * zpo);
  const int qd = warp & 3;  // TMEM lane quarter this warp may access
#pragma unroll 1
  for (int i = 0; i < 4; ++i) {
    const int mb = (NW == 8 ? (warp & 4) : 0) + i;  // M block (= producing warp)
    float vals[32];
    if (s_has[mb]) {
      const uint32_t ta = tmem_base + ((uint32_t)(qd * 32) << 16) + (uint32_t)(mb * kN);
      if (CM + 1 <= 20)
        tc::tmem_ld_32x32b_x20(ta, vals);  // classes + sigma only
      else
        tc::tmem_ld_32x32b_x32(ta, vals);
    } else {
#pragma unroll
      for (int k = 0; k < 32; ++k) vals[k] = 0.0f;
    }
    // TMEM lane 32*qd + lane = row = src_lane*4 + v of block mb
    const int src = qd * 8 + (lane >> 2), v = lane & 3;
    const int vx = (mb & 1) * 4 + (src & 3);
    const int vy = ((mb >> 1) & 1) * 4 + ((src >> 2) & 3);
    const int vz = (mb >> 2) * 8 + (src >> 4) * 4 + v;
    const int loc = vx + kTileX * vy;  // within the z layer
    int best = 0;
    float bv = vals[0];
    if (C == CM) {  // the usual case: no per-class bound test
#pragma unroll
      for (int k = 1; k < CM; ++k)
        if (vals[k] > bv) {
          bv = vals[k];
          best = k;
        }
    } else {
#pragma unroll
      for (int k = 1; k < CM; ++k)
        if (k < C && vals[k] > bv) {
          bv = vals[k];
          best = k;
        }
    }
    const float vo = vals[CM];
    if (A.v_c) {
      if ((CM & 1) == 0 && C == CM) {  // 8-byte stores: zpc and loc * C are even
        float2* d2 = reinterpret_cast<float2*>(s_vc + vz * zpc + loc * CM);
#pragma unroll
        for (int k = 0; k < CM / 2; ++k) d2[k] = make_float2(vals[2 * k], vals[2 * k + 1]);
      } else {
#pragma unroll
        for (int k = 0; k < CM; ++k)
          if (k < C) s_vc[vz * zpc + loc * C + k] = vals[k];
      }
    }
    s_vo[vz * zpo + loc] = vo;
    s_lab[vz * zpo + loc] = (vo < A.tau) ? (uint8_t)A.free_label : (uint8_t)best;
  }
  tc::fence_proxy_async_smem();  // staging -> visible to the bulk-copy engine
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  // rows of 8 voxels: warp w owns y rows y_t + RPW*w .. + RPW-1 for every z
  // layer; lane < 16 takes (row RPW*w + lane / LZ, layer lane % LZ)
  const int64_t V = (int64_t)nx * ny * nz;
  const int xw = min(kTileX, nx - x_t);
  const int zend = min(LZ, nz - z_t);
  const int64_t zstep = (int64_t)nx * ny;
  // Full rows whose global addresses are 16-byte aligned go out as bulk
  // async copies (one lane per (row, z layer): the v_c row of 8*C floats and
  // the v_o row of 8 floats) and one 8-byte label store; the rest take the
  // lane-parallel path.  Alignment is uniform per launch (row and layer
  // strides), so the choice is warp-uniform.
  const bool full = xw == kTileX;
  const bool vc_bulk = !A.v_c || (full && ((nx * C) & 3) == 0 && ((V * C) & 3) == 0 &&
                                  (reinterpret_cast<uintptr_t>(A.v_c) & 15) == 0);
  const bool vo_bulk = !A.v_o || (full && (nx & 3) == 0 && (V & 3) == 0 &&
                                  (reinterpret_cast<uintptr_t>(A.v_o) & 15) == 0);
  const bool lab8 = full && (nx & 7) == 0 && (V & 7) == 0 &&
                    (reinterpret_cast<uintptr_t>(A.labels) & 7) == 0;
  if (vc_bulk && vo_bulk && lab8) {
    // v_c rows (8*C floats) as bulk copies, one per (row, layer) lane; the
    // 32-byte v_o rows as two 16-byte lane stores each (all 32 lanes), the
    // 8-byte label rows as one lane store each
    {
      const int p = lane >> 1, half = lane & 1;
      const int ry = RPW * warp + p / LZ, zl = p % LZ;
      const int yy = y_t + ry;
      if (A.v_o && zl < zend && yy < ny) {
        const int64_t gv =
            (int64_t)f * V + (int64_t)x_t + (int64_t)nx * (yy + (int64_t)ny * (z_t + zl));
        *reinterpret_cast<float4*>(A.v_o + gv + half * 4) =
            *reinterpret_cast<const float4*>(s_vo + zl * zpo + ry * kTileX + half * 4);
      }
    }
    const int ry = RPW * warp + lane / LZ, zl = lane % LZ;
    const int yy = y_t + ry;
    if (lane < 16 && zl < zend && yy < ny) {
      const int64_t gv = (int64_t)f * V + (int64_t)x_t + (int64_t)nx * (yy + (int64_t)ny * (z_t + zl));
      if (A.v_c)
        tc::bulk_store(A.v_c + gv * C, tc::smem_u32(s_vc + zl * zpc + ry * kTileX * C),
                       (uint32_t)(kTileX * C * 4));
      *reinterpret_cast<uint2*>(A.labels + gv) =
          *reinterpret_cast<const uint2*>(s_lab + zl * zpo + ry * kTileX);
    }
    // commit + wait outside the per-lane issue (which the compiler runs as
    // a loop over lanes): all copies are in flight before any lane waits;
    // the staging must outlive their reads
    __syncwarp();
    tc::bulk_commit_wait_read();
  } else {
    const int nel = xw * C;
    const bool vec4 = (nel & 3) == 0 && ((kTileX * C) & 3) == 0;
    const int nel4 = nel >> 2;
#pragma unroll 1
    for (int r = 0; r < RPW; ++r) {
      const int ry = RPW * warp + r;
      const int yy = y_t + ry;
      if (yy >= ny) break;
      int64_t gv = (int64_t)f * V + (int64_t)x_t + (int64_t)nx * (yy + (int64_t)ny * z_t);
      for (int zl = 0; zl < zend; ++zl, gv += zstep) {
        if (A.v_c) {
          const float* src = s_vc + zl * zpc + ry * kTileX * C;  // 16-byte aligned
          float* dst = A.v_c + gv * C;
          if (vec4 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
            const float4* s4 = reinterpret_cast<const float4*>(src);
            float4* d4 = reinterpret_cast<float4*>(dst);
            for (int e = lane; e < nel4; e += 32) d4[e] = s4[e];
          } else {
            for (int e = lane; e < nel; e += 32) dst[e] = src[e];
          }
        }
        if (lane < xw) {
          if (A.v_o) A.v_o[gv + lane] = s_vo[zl * zpo + ry * kTileX + lane];
          A.labels[gv + lane] = s_lab[zl * zpo + ry * kTileX + lane];
        }
      }
    }
  }
}

template <int CM, int FIELD, bool PERSIST, int NW = 8>
__global__ void __launch_bounds__(NW * 32, 16 / NW) eval_tc_kernel(EvalArgs A) {
  using S = TcShape<CM, NW>;
  constexpr int kHalves = 8 / NW;  // CTAs per bin tile (NW = 4: one per z half)
  const int n_items = A.n_tiles * kHalves;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* s_rec = smem + S::kRec;
  uint16_t* s_list = reinterpret_cast<uint16_t*>(smem + S::kList);
  uint16_t* s_bm = reinterpret_cast<uint16_t*>(smem + S::kBm);
  uint8_t* s_acc = smem + S::kAcc;
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(smem + S::kBar);
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + S::kMisc);
  int* s_has = reinterpret_cast<int*>(smem + S::kMisc + 4);

  int* s_next = reinterpret_cast<int*>(smem + S::kMisc + 4 + NW * 4);
  if (!PERSIST) {
    const int tg = (int)blockIdx.x / kHalves;
    if (A.tile_off[tg + 1] - A.tile_off[tg] > A.tc_max_entries)
      return;  // a deep tile: the CUDA-core evaluator (launched next) owns it
  }
  // warp index and TMEM base through a lane-0 shuffle: provably warp-uniform
  // for ptxas, so the MMA operands derived from them live in uniform
  // registers (no per-issue elect/broadcast loops)
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);

  // ---- TMEM + barriers ----
  if (warp == 0) {
    tc::tmem_alloc(s_tmem, NW * kN);
    tc::tmem_relinquish();
  }
  if (lane == 0) tc::mbar_init(&s_bar[warp], 1);
  if (tid == 0) tc::fence_mbar_init();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *s_tmem, 0);
  const uint32_t d_tmem = tmem_base + (uint32_t)(warp * kN);

  uint8_t* a_hi = smem + S::kA + warp * 8192;
  uint8_t* a_lo = a_hi + 4096;
  uint8_t* b_hi = smem + S::kB + warp * 2048;
  uint8_t* b_lo = b_hi + 1024;
  // MN-major BASE32B: A 128 rows (LBO 512, SBO 2048), B 32 rows (LBO 512, SBO 512)
  const uint64_t da_hi = tc::smem_desc_mn32(tc::smem_u32(a_hi), 512, 2048);
  const uint64_t da_lo = tc::smem_desc_mn32(tc::smem_u32(a_lo), 512, 2048);
  const uint64_t db_hi = tc::smem_desc_mn32(tc::smem_u32(b_hi), 512, 512);
  const uint64_t db_lo = tc::smem_desc_mn32(tc::smem_u32(b_lo), 512, 512);

  int kk = 0;            // primitives in the open K step
  int groups = 0;        // K steps issued by this warp
  uint32_t phase = 0;    // parity of the next mbarrier completion to wait for
  bool pending = false;  // an issued K step not yet known complete

  auto wait_free = [&]() {
    if (pending) {
      tc::mbar_wait(&s_bar[warp], phase);
      phase ^= 1u;
      pending = false;
    }
  };

  // primitive in K slot k: A rows lane*4 + v (one STS.128), B row lane
  // per-lane parts of the operand offsets (tc::mn32_offset with mn = lane*4
  // for A, mn = lane for B); the K slot adds a uniform part and a swizzle XOR
  // The lane parts (bits 2-6, 9-10) and the K-slot parts (bits 7-8, 9 or 11)
  // occupy disjoint bits except the swizzle bits 5-6, so offset = lane ^ slot.
  const uint32_t a_lane = (uint32_t)((lane >> 3) * 512 + (lane & 1) * 16) |
                          (uint32_t)(((lane >> 1) & 3) << 5);
  const uint32_t b_lane = (uint32_t)((lane & 7) * 4) | (uint32_t)(((lane >> 3) & 3) << 5);
  auto store_k = [&](int k, const float(&w)[kVPT], float cw) {
    // slot part: (k & 3) * 160 | (k >> 2) << 11 (A), << 9 (B), as sums
    const uint32_t k160 = (uint32_t)k * 160u, k4 = (uint32_t)(k & 4);
    const uint32_t ao = a_lane ^ (k160 + k4 * 352u);
    const uint32_t bo = b_lane ^ (k160 - k4 * 32u);
    float4 h, l;
    h.x = tf32_hi(w[0]);
    h.y = tf32_hi(w[1]);
    h.z = tf32_hi(w[2]);
    h.w = tf32_hi(w[3]);
    l.x = w[0] - h.x;
    l.y = w[1] - h.y;
    l.z = w[2] - h.z;
    l.w = w[3] - h.w;
    *reinterpret_cast<float4*>(a_hi + ao) = h;
    *reinterpret_cast<float4*>(a_lo + ao) = l;
    const float ch = tf32_hi(cw);
    *reinterpret_cast<float*>(b_hi + bo) = ch;
    *reinterpret_cast<float*>(b_lo + bo) = cw - ch;
  };
  auto issue = [&]() {
    tc::fence_proxy_async_smem();
    __syncwarp();
    tc::fence_after_sync();
    tc::mma3_tf32_commit(d_tmem, da_hi, da_lo, db_hi, db_lo, kIdesc, groups == 0 ? 1u : 0u,
                         &s_bar[warp]);
    __syncwarp();
    ++groups;
    pending = true;
    kk = 0;
  };
  // ---- persistent loop over tiles: tile 0 of this CTA is blockIdx.x, the
  // rest come from a global counter (dynamic balance; tiles vary from 0 to
  // hundreds of primitives).  TMEM, barriers and descriptors are set up once;
  // the first chunk of the next tile is staged (cp.async) while the epilogue
  // of the current one runs when the epilogue staging leaves s_rec alone.
  constexpr bool kPrefetch = S::kStage <= S::kRec;
  constexpr bool kSplitAcc = FIELD == 6;
  auto stage_chunk = [&](int64_t fb, int c0, int n) {
    // two threads per primitive, every 16-byte piece in flight at once
    static_assert(2 * S::kChunk <= NW * 32, "staging map");
    const int j = tid >> 1;
    if (j < n) {
      if ((tid & 1) == 0) s_bm[j] = (uint16_t)A.bmask[c0 + j];
      const int64_t g = fb + A.prim_ids[c0 + j];
      const float4* rsrc = reinterpret_cast<const float4*>(A.recs + g * kRecWords);
      const float4* lsrc = reinterpret_cast<const float4*>(A.lrows + g * A.lrow);
      const uint32_t dst = tc::smem_u32(s_rec + j * S::kStride * 4);
#pragma unroll
      for (int q = tid & 1; q < S::kStride / 4; q += 2)
        tc::cp_async16(dst + q * 16, q < kRecWords / 4 ? rsrc + q : lsrc + (q - kRecWords / 4));
    }
  };
  int item = blockIdx.x;
  bool prefetched = false;
  while (item < n_items) {
    const int tile_g = item / kHalves, half = item - tile_g * kHalves;
    const int blk = half * NW + warp;  // this warp's block of the bin tile (mask bit)
    const int f = tile_g / A.tiles_per_frame;
    const int t = tile_g - f * A.tiles_per_frame;
    const int tx = t % A.ntx;
    const int ty = (t / A.ntx) % A.nty;
    const int tz = t / (A.ntx * A.nty);
    const int bx0 = tx * kTileX + (blk & 1) * 4;
    const int by0 = ty * kTileY + ((blk >> 1) & 1) * 4;
    const int bz0 = tz * kTileZ + (blk >> 2) * 8;
    const int x = bx0 + (lane & 3);
    const int y = by0 + ((lane >> 2) & 3);
    const int z0 = bz0 + (lane >> 4) * 4;
    kk = 0;
    groups = 0;
    // claim the next tile now; the result is only needed at the epilogue
    const int claimed = (PERSIST && tid == 0) ? atomicAdd(A.tile_counter, 1) : 0;
    const int beg = A.tile_off[tile_g];
    int end = A.tile_off[tile_g + 1];
    // a deep tile is left to the CUDA-core evaluator (launched next, which
    // overwrites the zeros written here)
    if (end - beg > A.tc_max_entries) end = beg;
    const int64_t fbase = (int64_t)f * A.n_prims;
    for (int c0 = beg; c0 < end; c0 += S::kChunk) {
      const int n = min(S::kChunk, end - c0);
      if (!(prefetched && c0 == beg)) {
        __syncthreads();  // every warp is done with the previous chunk
        stage_chunk(fbase, c0, n);
      }
      tc::cp_async_wait_all();
      __syncthreads();
      uint16_t* lst = s_list + warp * S::kChunk;
      uint8_t* lst_acc = s_acc + warp * S::kChunk;
      int n_in = 0, n_part = 0, n_acc = 0;  // warp-uniform list lengths
      const unsigned lt = (1u << lane) - 1u;
      for (int q = 0; q * 32 < n; ++q) {
        const int j = q * 32 + lane;
        // this warp's bits of the precomputed block masks (block_masks_kernel)
        const unsigned m = j < n ? (unsigned)s_bm[j] : 0u;
        bool hit = (m >> blk) & 1u, inside = (m >> (8 + blk)) & 1u;
        if (kSplitAcc) {  // strict: accurate-log primitives get their own list
          const bool acc =
              hit && reinterpret_cast<const PrimRec*>(s_rec + j * S::kStride * 4)->c > SQV_ACC_C;
          const unsigned ma = __ballot_sync(0xffffffffu, acc);
          if (acc) lst_acc[n_acc + __popc(ma & lt)] = (uint8_t)j;
          n_acc += __popc(ma);
          hit &= !acc;
          inside &= !acc;
        }
        const unsigned mi = __ballot_sync(0xffffffffu, inside);
        const unsigned mp = __ballot_sync(0xffffffffu, hit && !inside);
        const uint16_t off = (uint16_t)(j * (S::kStride / 4));  // 16-byte units
        if (inside) lst[n_in + __popc(mi & lt)] = off;
        if (hit && !inside) lst[S::kChunk - 1 - (n_part + __popc(mp & lt))] = off;
        n_in += __popc(mi);
        n_part += __popc(mp);
      }
      __syncwarp();
      if (lane == 0)
        add_stats(A.stats, (n_in + n_part) * mufu_per_block(FIELD, false) +
                               n_acc * mufu_per_block(FIELD, true), n_in + n_part + n_acc);
      // the operands are single-buffered: a K step's MMAs must complete
      // before the next primitive's stores.  Both modes wait right after the
      // issue (round 1 had strict wait right before the next stores, +0.8%
      // then; with the folded exponents of round 2 the early wait is +0.6%
      // on config 1)
      constexpr bool kLateWait = false;
      auto push = [&](const float(&w)[kVPT], float cw) {
        if (kLateWait) wait_free();
        store_k(kk, w, cw);
        if (++kk == kK) {
          issue();
          if (!kLateWait) wait_free();
        }
      };
      // class weight n = lane (sigma at CM), zero beyond
      auto class_weight = [&](int off) {
        return lane < S::kLRow ? reinterpret_cast<const float*>(s_rec + off + kRecWords * 4)[lane]
                               : 0.0f;
      };
      // whole-block primitives first (no per-voxel window test), then the rest,
      // each in ascending primitive order
      const int n_tot = n_in + n_part;
      auto off_at = [&](int k) {
        return (int)(k < n_in ? lst[k] : lst[S::kChunk - 1 - (k - n_in)]) << 4;
      };
      if constexpr (FIELD == 6 || FIELD == 7) {
        // two-stage software pipeline: the logs of primitive k interleave with
        // the exps of primitive k-1 (independent chains for the latency-bound
        // SFU/FMA mix); the hand-off lives in registers
        // One pipelined pass over a list (whole-block primitives, LIVE =
        // false, or partial ones, LIVE = true): no per-primitive branch on
        // the list kind.  Strict mode has already moved its accurate-log
        // primitives to lst_acc; fast mode has none.
        auto run = [&](auto live, int cnt, auto off_of) {
          constexpr bool LIVE = decltype(live)::value;
          if (cnt <= 0) return;
          // (strict mode's accurate-log primitives are in lst_acc, so every
          // primitive here takes the SFU logs: the step has no branch)
          auto step = [&](int off, PairState& nxt, const PairState& cur, float(&w)[kVPT]) {
            const PrimRec& R = *reinterpret_cast<const PrimRec*>(s_rec + off);
            nxt.cw = class_weight(off);
            stage_exps<true>(cur, w);
            stage_logs<FIELD == 6, LIVE, false>(R, x, y, z0, nxt);
          };
          PairState s0, s1;
          float w[kVPT];
          {
            const int off = off_of(0);
            const PrimRec& R = *reinterpret_cast<const PrimRec*>(s_rec + off);
            s0.cw = class_weight(off);
            stage_logs<FIELD == 6, LIVE, false>(R, x, y, z0, s0);
          }
          // an even K slot at the loop head lets each two-primitive iteration
          // check for a full K step once (pad with a zero column if odd)
          if (kk & 1) {
            const float zw[kVPT] = {0.f, 0.f, 0.f, 0.f};
            push(zw, 0.0f);
          }
          // list entries are read one step ahead (past the end: harmless
          // reads inside the CTA's shared memory, discarded)
          int k = 1, off = off_of(1);
          for (; k + 1 < cnt; k += 2) {  // ping-pong: no state copies
            const int off1 = off_of(k + 1);
            step(off, s1, s0, w);
            if (kLateWait) wait_free();  // the K step issued below, one iteration back
            store_k(kk++, w, s0.cw);     // kk odd after this: the step cannot be full
            off = off_of(k + 2);
            step(off1, s0, s1, w);
            store_k(kk++, w, s1.cw);
            if (kk == kK) {
              issue();
              if (!kLateWait) wait_free();
            }
          }
          if (k < cnt) {
            step(off, s1, s0, w);
            push(w, s0.cw);
            stage_exps<true>(s1, w);
            push(w, s1.cw);
          } else {
            stage_exps<true>(s0, w);
            push(w, s0.cw);
          }
        };
        run(std::false_type{}, n_in, [&](int k) { return (int)lst[k] << 4; });
        run(std::true_type{}, n_part, [&](int k) { return (int)lst[S::kChunk - 1 - k] << 4; });
        // strict: the accurate-log primitives after the rest, unpipelined
        // (their long FMA-pipe logs no longer double the pipelined loop's code)
        if (kSplitAcc)
          for (int k = 0; k < n_acc; ++k) {
            const int off = (int)lst_acc[k] * S::kStride * 4;
            const PrimRec& R = *reinterpret_cast<const PrimRec*>(s_rec + off);
            PairState st;
            float w[kVPT];
            stage_logs<true, true, true>(R, x, y, z0, st);  // exact steps, window test, acc logs
            stage_exps<true>(st, w);
            push(w, class_weight(off));
          }
      } else {
        for (int k = 0; k < n_tot; ++k) {
          const int off = off_at(k);
          const PrimRec& R = *reinterpret_cast<const PrimRec*>(s_rec + off);
          float w[kVPT];
          pair_weights<FIELD, true>(R, x, y, z0, w);
          push(w, class_weight(off));
        }
      }
    }
    if (kk > 0) {  // close the last K step with zero columns
      const float zw[kVPT] = {0.f, 0.f, 0.f, 0.f};
      wait_free();
      for (int k = kk; k < kK; ++k) store_k(k, zw, 0.0f);
      issue();
    }
    wait_free();
    if (lane == 0) s_has[warp] = groups > 0;
    // next tile (one atomic per CTA), published by the barrier below
    if (PERSIST && tid == 0) *s_next = (int)gridDim.x + claimed;
    tc::fence_before_sync();
    __syncthreads();  // all MMAs complete; operand smem is free for staging
    tc::fence_after_sync();
    const int next_item = PERSIST ? *s_next : n_items;
    prefetched = false;
    if (PERSIST && kPrefetch && next_item < n_items) {
      const int ntg = next_item / kHalves;
      const int nb = A.tile_off[ntg], ne = A.tile_off[ntg + 1];
      if (ne > nb && ne - nb <= A.tc_max_entries) {
        const int nf = ntg / A.tiles_per_frame;
        stage_chunk((int64_t)nf * A.n_prims, nb, min(S::kChunk, ne - nb));
        prefetched = true;
      }
    }

    tile_epilogue<CM, NW>(A, smem, s_has, tmem_base, warp, lane, f, tx, ty, tz, half * 8);

    // all TMEM reads and bulk-copy reads of the staging are done before the
    // next item's MMAs and operand stores reuse them
    if (PERSIST && next_item < n_items) {
      tc::fence_before_sync();
      __syncthreads();
      tc::fence_after_sync();
    }
    item = next_item;
  }  // item loop
  if (warp == 0) tc::tmem_dealloc(tmem_base, NW * kN);
}


// ---- streaming variant: per-warp lists and per-warp staging rings -------
//
// No CTA barrier inside a tile.  Each warp builds its own hit lists for a
// segment of the tile's entries straight from the block masks in global
// memory (bit 16 = strict mode's accurate-log primitives), then streams the
// records of its hits through a private shared-memory ring with cp.async,
// issued a few primitives ahead of use.  A warp with fewer hits never waits
// for the others before the tile's epilogue, and no warp waits for a
// CTA-wide chunk to land.  Same per-pair math, K-step packing and epilogue
// as eval_tc_kernel.
#ifndef SQV_RING
#define SQV_RING 8
#endif
#ifndef SQV_SEG
#define SQV_SEG 256
#endif
template <int CM, int NW>
struct TcsShape {
  static constexpr int kLRow = (CM + 1 + 3) & ~3;
  static constexpr int kStride = kRecWords + kLRow;  // words per staged primitive
  static constexpr int kPieces = kStride / 4;        // 16-byte copies per primitive
  static constexpr int kD = SQV_RING;                // ring slots per warp
  static_assert((kD & (kD - 1)) == 0 && kD >= 4, "ring slots: a power of two >= 4");
  static constexpr int kSeg = SQV_SEG;               // entries per list segment
  static_assert(kSeg % 32 == 0, "segments of whole ballots");
  static constexpr int kA = 0;
  static constexpr int kB = kA + NW * 2 * 4096;
  static constexpr int kRing = kB + NW * 2 * 1024;
  static constexpr int kList = kRing + NW * kD * kStride * 4;
  static constexpr int kBar = (kList + NW * kSeg * 4 + 7) & ~7;
  static constexpr int kMisc = kBar + NW * 8;        // tmem base + has flags + next tile
  static constexpr int kEnd = kMisc + 4 + NW * 4 + 4;
  static constexpr int kStage = 2 * NW * ((64 * CM + 8) * 4 + 72 * 4 + 72);
  static_assert(kStage <= kBar, "epilogue staging must not reach the barriers");
  static constexpr int kBody = kEnd > kStage ? kEnd : kStage;
  static constexpr int kSmem = kBody + 1024;
  static constexpr int kCtasPerSm = 16 / NW;         // 16 warp blocks of TMEM per SM
  static_assert(kCtasPerSm * (kSmem + 1024) <= 228 * 1024, "CTAs per SM by shared memory");
};

// NW = 8: one CTA per 8x8x16 bin tile, two per SM.  NW = 4: one CTA per z
// half of a bin tile (warp blocks 4h..4h+3 of its masks), four per SM: a
// CTA's tile-end barrier and epilogue idle a quarter of the SM's warps
// instead of half.
template <int CM, int FIELD, bool PERSIST, int NW>
__global__ void __launch_bounds__(NW * 32, 16 / NW) eval_tcs_kernel(EvalArgs A) {
  using S = TcsShape<CM, NW>;
  constexpr int kHalves = 8 / NW;  // CTAs per bin tile
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(smem + S::kBar);
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + S::kMisc);
  int* s_has = reinterpret_cast<int*>(smem + S::kMisc + 4);
  int* s_next = reinterpret_cast<int*>(smem + S::kMisc + 4 + NW * 4);
  const int n_items = A.n_tiles * kHalves;  // (bin tile, z half) work items
  if (!PERSIST) {
    const int tg = (int)blockIdx.x / kHalves;
    if (A.tile_off[tg + 1] - A.tile_off[tg] > A.tc_max_entries)
      return;  // a deep tile: the CUDA-core evaluator (launched next) owns it
  }
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);

  if (warp == 0) {
    tc::tmem_alloc(s_tmem, NW * kN);
    tc::tmem_relinquish();
  }
  if (lane == 0) tc::mbar_init(&s_bar[warp], 1);
  if (tid == 0) tc::fence_mbar_init();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *s_tmem, 0);
  const uint32_t d_tmem = tmem_base + (uint32_t)(warp * kN);

  uint8_t* a_hi = smem + S::kA + warp * 8192;
  uint8_t* a_lo = a_hi + 4096;
  uint8_t* b_hi = smem + S::kB + warp * 2048;
  uint8_t* b_lo = b_hi + 1024;
  const uint64_t da_hi = tc::smem_desc_mn32(tc::smem_u32(a_hi), 512, 2048);
  const uint64_t da_lo = tc::smem_desc_mn32(tc::smem_u32(a_lo), 512, 2048);
  const uint64_t db_hi = tc::smem_desc_mn32(tc::smem_u32(b_hi), 512, 512);
  const uint64_t db_lo = tc::smem_desc_mn32(tc::smem_u32(b_lo), 512, 512);
  // this warp's staging ring and sequence list
  uint8_t* ring = smem + S::kRing + warp * (S::kD * S::kStride * 4);
  const uint32_t ring_s = tc::smem_u32(ring);
  int* wl = reinterpret_cast<int*>(smem + S::kList) + warp * S::kSeg;

  int kk = 0, groups = 0;
  uint32_t phase = 0;
  bool pending = false;
  auto wait_free = [&]() {
    if (pending) {
      tc::mbar_wait(&s_bar[warp], phase);
      phase ^= 1u;
      pending = false;
    }
  };
  const uint32_t a_lane = (uint32_t)((lane >> 3) * 512 + (lane & 1) * 16) |
                          (uint32_t)(((lane >> 1) & 3) << 5);
  const uint32_t b_lane = (uint32_t)((lane & 7) * 4) | (uint32_t)(((lane >> 3) & 3) << 5);
  auto store_k = [&](int k, const float(&w)[kVPT], float cw) {
    const uint32_t k160 = (uint32_t)k * 160u, k4 = (uint32_t)(k & 4);
    const uint32_t ao = a_lane ^ (k160 + k4 * 352u);
    const uint32_t bo = b_lane ^ (k160 - k4 * 32u);
    float4 h, l;
    h.x = tf32_hi(w[0]);
    h.y = tf32_hi(w[1]);
    h.z = tf32_hi(w[2]);
    h.w = tf32_hi(w[3]);
    l.x = w[0] - h.x;
    l.y = w[1] - h.y;
    l.z = w[2] - h.z;
    l.w = w[3] - h.w;
    *reinterpret_cast<float4*>(a_hi + ao) = h;
    *reinterpret_cast<float4*>(a_lo + ao) = l;
    const float ch = tf32_hi(cw);
    *reinterpret_cast<float*>(b_hi + bo) = ch;
    *reinterpret_cast<float*>(b_lo + bo) = cw - ch;
  };
  auto issue = [&]() {
    tc::fence_proxy_async_smem();
    __syncwarp();
    tc::fence_after_sync();
    tc::mma3_tf32_commit(d_tmem, da_hi, da_lo, db_hi, db_lo, kIdesc, groups == 0 ? 1u : 0u,
                         &s_bar[warp]);
    __syncwarp();
    ++groups;
    pending = true;
    kk = 0;
  };
  constexpr bool kSplitAcc = FIELD == 6;
  // a K step's MMAs are waited for right after their issue in both modes
  // (strict waiting before the next stores instead, as the chunk-staged
  // kernel does, measured 1.6% slower here)
  constexpr bool kLateWait = false;
  constexpr int kSlotBytes = S::kStride * 4;
  // per-lane constants of the ring copies: lane -> (item within a round of
  // kItemsPerRound items, 16-byte piece); the source of a piece is
  // cp_src + (primitive record index) * cp_mult
  constexpr int kItemsPerRound = 32 / S::kPieces;
  static_assert(kItemsPerRound >= 1, "a primitive's pieces fit one warp");
  constexpr int kCopyRounds = (S::kD / 2 + kItemsPerRound - 1) / kItemsPerRound;
  const int cp_item = lane / S::kPieces, cp_pc = lane - cp_item * S::kPieces;
  const bool cp_live = cp_item < kItemsPerRound;
  const uint32_t cp_dst = (uint32_t)(cp_pc * 16);
  const char* cp_src = cp_pc < kRecWords / 4
                           ? reinterpret_cast<const char*>(A.recs) + cp_pc * 16
                           : reinterpret_cast<const char*>(A.lrows) + (cp_pc - kRecWords / 4) * 16;
  const int cp_mult = cp_pc < kRecWords / 4 ? kRecWords * 4 : A.lrow * 4;

  int item = blockIdx.x;
  while (item < n_items) {
    const int tile_g = item / kHalves, half = item - tile_g * kHalves;
    const int blk = half * NW + warp;  // this warp's block of the bin tile (mask bit)
    const int f = tile_g / A.tiles_per_frame;
    const int t = tile_g - f * A.tiles_per_frame;
    const int tx = t % A.ntx;
    const int ty = (t / A.ntx) % A.nty;
    const int tz = t / (A.ntx * A.nty);
    const int x = tx * kTileX + (blk & 1) * 4 + (lane & 3);
    const int y = ty * kTileY + ((blk >> 1) & 1) * 4 + ((lane >> 2) & 3);
    const int z0 = tz * kTileZ + (blk >> 2) * 8 + (lane >> 4) * 4;
    kk = 0;
    groups = 0;
    const int claimed = (PERSIST && tid == 0) ? atomicAdd(A.tile_counter, 1) : 0;
    const int beg = A.tile_off[tile_g];
    int end = A.tile_off[tile_g + 1];
    if (end - beg > A.tc_max_entries) end = beg;
    const int fbase = f * A.n_prims;
#ifdef SQV_DIAG_IMBAL
    int diag_items = 0;
#endif
    for (int c0 = beg; c0 < end; c0 += S::kSeg) {
      const int n = min(S::kSeg, end - c0);
      // ---- this warp's sequence of the segment, from the block masks:
      // whole-block hits, then partial ones, then (strict) accurate-log ones,
      // each in ascending entry order; two passes over the ballots (counts,
      // then positions), so the sequence is one contiguous array ----
      int n_in = 0, n_part = 0, n_acc = 0;  // warp-uniform
      {
        constexpr int kQ = S::kSeg / 32;
        unsigned bi[kQ], bp[kQ], ba[kQ], mq[kQ];
        int gq[kQ];
#pragma unroll
        for (int q = 0; q < kQ; ++q) {  // every load in flight at once
          const int j = q * 32 + lane;
          mq[q] = j < n ? __ldg(A.bmask + c0 + j) : 0u;
          gq[q] = j < n ? __ldg(A.prim_ids + c0 + j) : 0;
        }
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
          if (q * 32 >= n) break;
          const unsigned m = mq[q];
          const bool hit = (m >> blk) & 1u, inside = (m >> (8 + blk)) & 1u;
          const bool acc = kSplitAcc && hit && ((m >> 16) & 1u);
          ba[q] = __ballot_sync(0xffffffffu, acc);
          bi[q] = __ballot_sync(0xffffffffu, inside && !acc);
          bp[q] = __ballot_sync(0xffffffffu, hit && !inside && !acc);
          n_in += __popc(bi[q]);
          n_part += __popc(bp[q]);
          n_acc += __popc(ba[q]);
        }
        const unsigned lt = (1u << lane) - 1u, me = 1u << lane;
        int oi = 0, op = n_in, oa = n_in + n_part;
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
          if (q * 32 >= n) break;
          if (bi[q] & me) wl[oi + __popc(bi[q] & lt)] = gq[q];
          if (bp[q] & me) wl[op + __popc(bp[q] & lt)] = gq[q];
          if (ba[q] & me) wl[oa + __popc(ba[q] & lt)] = gq[q];
          oi += __popc(bi[q]);
          op += __popc(bp[q]);
          oa += __popc(ba[q]);
        }
        __syncwarp();
      }
      // ---- the ring: sequence item q lives in slot q % kD; items are copied
      // in batches of half a ring (one cp.async group); batch b is waited for
      // right before its first item is read, and batch b+1 is issued once
      // batch b-1 has been read (its half of the ring is free) ----
      const int n_seq = n_in + n_part + n_acc;
#ifdef SQV_DIAG_IMBAL
      diag_items += n_seq;
#endif
      if (lane == 0)
        add_stats(A.stats, (n_in + n_part) * mufu_per_block(FIELD, false) +
                               n_acc * mufu_per_block(FIELD, true), n_seq);
      constexpr int kH = S::kD / 2;           // items per batch
      int issued = 0;                          // batches issued
      auto copy_batch = [&](int bt) {
#pragma unroll
        for (int r = 0; r < kCopyRounds; ++r) {
          const int q = bt * kH + r * kItemsPerRound + cp_item;
          if (cp_live && r * kItemsPerRound + cp_item < kH && q < n_seq)
            tc::cp_async16(ring_s + (uint32_t)((q & (S::kD - 1)) * kSlotBytes) + cp_dst,
                           cp_src + (int64_t)(fbase + wl[q]) * cp_mult);
        }
        tc::cp_async_commit();
      };
      int wmark = 0, rmark = kH;
      // items < qlo are read (their slots are free); items up to qhi are
      // about to be read
      auto feed = [&](int qlo, int qhi) {
        if (qlo >= rmark) {  // batch rmark/kH - 1 is read: its half takes batch rmark/kH + 1
          if (rmark + kH < n_seq) {
            copy_batch(rmark / kH + 1);
            ++issued;
          }
          rmark += kH;
        }
        if (qhi >= wmark) {  // first read of batch wmark/kH: wait for it
          if (issued - 1 > wmark / kH)
            tc::cp_async_wait_group<1>();
          else
            tc::cp_async_wait_group<0>();
          __syncwarp();
          wmark += kH;
        }
      };
      if (n_seq > 0) {
        copy_batch(0);
        issued = 1;
      }
      if (kH < n_seq) {
        copy_batch(1);
        issued = 2;
      }
      auto slot = [&](int q) { return ring + (q & (S::kD - 1)) * kSlotBytes; };
      auto push = [&](const float(&w)[kVPT], float cw) {
        if (kLateWait) wait_free();
        store_k(kk, w, cw);
        if (++kk == kK) {
          issue();
          if (!kLateWait) wait_free();
        }
      };
      auto class_weight = [&](const uint8_t* rec) {
        return lane < S::kLRow ? reinterpret_cast<const float*>(rec + kRecWords * 4)[lane] : 0.0f;
      };
      // one branch-free pipelined pass over the items [base, base + cnt) of
      // one kind (whole-block: LIVE = false; partial: LIVE = true)
      auto run = [&](auto live, int base, int cnt) {
        constexpr bool LIVE = decltype(live)::value;
        if (cnt <= 0) return;
        auto step = [&](int q, PairState& nxt, const PairState& cur, float(&w)[kVPT]) {
          const uint8_t* rec = slot(q);
          const PrimRec& R = *reinterpret_cast<const PrimRec*>(rec);
          nxt.cw = class_weight(rec);
          stage_exps<true>(cur, w);
          stage_logs<FIELD == 6, LIVE, false>(R, x, y, z0, nxt);
        };
        PairState s0, s1;
        float w[kVPT];
        feed(base, base);
        {
          const uint8_t* rec = slot(base);
          s0.cw = class_weight(rec);
          stage_logs<FIELD == 6, LIVE, false>(*reinterpret_cast<const PrimRec*>(rec), x, y, z0, s0);
        }
        if (kk & 1) {
          const float zw[kVPT] = {0.f, 0.f, 0.f, 0.f};
          push(zw, 0.0f);
        }
        int k = 1;
        for (; k + 1 < cnt; k += 2) {
          feed(base + k, base + k + 1);
          step(base + k, s1, s0, w);
          if (kLateWait) wait_free();
          store_k(kk++, w, s0.cw);
          step(base + k + 1, s0, s1, w);
          store_k(kk++, w, s1.cw);
          if (kk == kK) {
            issue();
            if (!kLateWait) wait_free();
          }
        }
        if (k < cnt) {
          feed(base + k, base + k);
          step(base + k, s1, s0, w);
          push(w, s0.cw);
          stage_exps<true>(s1, w);
          push(w, s1.cw);
        } else {
          stage_exps<true>(s0, w);
          push(w, s0.cw);
        }
      };
      run(std::false_type{}, 0, n_in);
      run(std::true_type{}, n_in, n_part);
      if (kSplitAcc)  // strict: the accurate-log primitives, unpipelined
        for (int k = 0; k < n_acc; ++k) {
          const int q = n_in + n_part + k;
          feed(q, q);
          const uint8_t* rec = slot(q);
          PairState st;
          float w[kVPT];
          stage_logs<true, true, true>(*reinterpret_cast<const PrimRec*>(rec), x, y, z0, st);
          stage_exps<true>(st, w);
          push(w, class_weight(rec));
        }
      __syncwarp();  // every slot read before the next segment refills the ring
    }
    if (kk > 0) {
      const float zw[kVPT] = {0.f, 0.f, 0.f, 0.f};
      wait_free();
      for (int k = kk; k < kK; ++k) store_k(k, zw, 0.0f);
      issue();
    }
    wait_free();
    if (lane == 0) s_has[warp] = groups > 0;
    if (PERSIST && tid == 0) *s_next = (int)gridDim.x + claimed;
#ifdef SQV_DIAG_IMBAL  // diagnostics: stats[2] += max over warps, stats[3] += sum
    __shared__ int s_diag[NW];
    if (lane == 0) s_diag[warp] = diag_items;
#endif
    tc::fence_before_sync();
    __syncthreads();  // all MMAs complete; operand smem is free for staging
    tc::fence_after_sync();
#ifdef SQV_DIAG_IMBAL
    if (tid == 0 && A.stats) {
      int mx = 0, sm = 0;
      for (int w = 0; w < NW; ++w) mx = max(mx, s_diag[w]), sm += s_diag[w];
      atomicAdd(A.stats + 2, (unsigned long long)mx);
      atomicAdd(A.stats + 3, (unsigned long long)sm);
    }
#endif
    const int next_item = PERSIST ? *s_next : n_items;
    tile_epilogue<CM, NW>(A, smem, s_has, tmem_base, warp, lane, f, tx, ty, tz, half * 8);
    if (PERSIST && next_item < n_items) {
      tc::fence_before_sync();
      __syncthreads();
      tc::fence_after_sync();
    }
    item = next_item;
  }
  if (warp == 0) tc::tmem_dealloc(tmem_base, NW * kN);
}

}  // namespace

template <int CM>
int launch_tc(const EvalArgs& A, int n_tiles, int field, cudaStream_t s) {
  using S = TcShape<CM>;
  // TMEM: 512 columns per SM, 32 per warp block.  Shared memory caps the
  // chunk-staged kernel and the 8-warp streaming one at two CTAs per SM
  // (>= 80 KB each) and the 4-warp streaming one at four.
  constexpr int smem_chunk = S::kSmem > 80 * 1024 ? S::kSmem : 80 * 1024;
  constexpr int smem_s4 = TcsShape<CM, 4>::kSmem > 46 * 1024 ? TcsShape<CM, 4>::kSmem : 46 * 1024;
  static int n_sm = 0;
  if (!n_sm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    if (n_sm < 1) n_sm = 148;
  }
  const bool pipelined = field == 6 || field == 7;
  bool persist = pipelined && A.tile_counter &&
                 A.n_entries < (int64_t)kPersistentBelow * n_tiles && n_tiles > 2 * n_sm;
  if (const char* pe = std::getenv("SQV_PERSIST"))  // tests / A-B: force 0 or 1
    persist = pipelined && A.tile_counter && std::atoi(pe) != 0;
  // Dense batches: the streaming kernel, 4 warps per CTA (config 2 +0.5%
  // strict / +1.5% fast, config 3 +3% over the chunk-staged one); sparse
  // (persistent) batches: the chunk-staged kernel (config 1 strict: streaming
  // 12% slower, its per-warp list build and first copies sit in the L2
  // latency of every small tile).  SQV_STREAM=0/1 forces either (A/B).
  int mode = pipelined && !persist ? 4 : 0;
  // (two work items per bin tile: keep the item index in int range)
  const bool stream_ok = n_tiles < (1 << 30);
  if (const char* se = std::getenv("SQV_STREAM")) mode = pipelined && std::atoi(se) != 0 ? 4 : 0;
  if (!stream_ok) mode = 0;
  void (*kern)(EvalArgs);
  int smem_bytes, threads, ctas_per_sm, items;
  if (mode == 4) {
    kern = field == 6 ? (persist ? eval_tcs_kernel<CM, 6, true, 4> : eval_tcs_kernel<CM, 6, false, 4>)
                      : (persist ? eval_tcs_kernel<CM, 7, true, 4> : eval_tcs_kernel<CM, 7, false, 4>);
    smem_bytes = smem_s4, threads = 128, ctas_per_sm = 4, items = 2 * n_tiles;
  } else {
    kern = field == 9   ? eval_tc_kernel<CM, 9, false>
           : field == 8 ? eval_tc_kernel<CM, 8, false>
           : field == 6 ? (persist ? eval_tc_kernel<CM, 6, true> : eval_tc_kernel<CM, 6, false>)
                        : (persist ? eval_tc_kernel<CM, 7, true> : eval_tc_kernel<CM, 7, false>);
    smem_bytes = smem_chunk, threads = kThreads, ctas_per_sm = 2, items = n_tiles;
  }
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes) !=
      cudaSuccess)
    return check_launch("eval_tc_kernel attribute");
  // Sparse tiles (few primitives each: per-tile setup, staging latency and
  // epilogue dominate) run persistent, work items handed out by
  // A.tile_counter; dense tiles run one CTA per work item.
  const int grid = persist ? ctas_per_sm * n_sm : items;
  if (grid < 1) return SQV_OK;
  kern<<<grid, threads, smem_bytes, s>>>(A);
  count_launch();
  return check_launch("eval_tc_kernel");
}

}  // namespace sqv
