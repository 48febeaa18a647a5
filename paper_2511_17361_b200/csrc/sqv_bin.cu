// sqv_bin.cu — per-frame binning: tile lists, tile offsets and block masks of
// a batch in one kernel, one CTA per frame.
//
// The bins are the (tile, primitive) entries of SPEC.md:385's coarse grid,
// each tile's primitives in ascending id (bit-identical to the oracle's bins
// and to the emit + radix-sort path in sqv_prep.cu / sqv_sort.cu, which stays
// for grids whose tile counters do not fit shared memory).  A frame's entries
// are contiguous (its base is the sum of the earlier frames' entry counts,
// accumulated by prep), so the sort only has to order a frame's entries by
// tile, stably in primitive order — a counting sort in shared memory:
//
//   1. count: the CTA's 8 warps take contiguous eighths of the frame's
//      primitives; each primitive adds 1 to each tile of its window's tile
//      rectangle in its warp's counter row (shared-memory atomics);
//   2. per tile, an exclusive prefix over the 8 rows gives each warp's first
//      rank in the tile, and the row total the tile's count; an exclusive
//      scan of the counts gives the tile offsets (tile_off) and the deep-tile
//      list of the CUDA-core complement;
//   3. scatter: each warp walks its primitives in order (windows read 32 at a
//      time and broadcast by shuffle), its lanes spread over the primitive's
//      tiles, and writes the entry at base + tile offset + the warp's running
//      rank in that tile: every tile lists its primitives in ascending id;
//   4. block masks: the CTA evaluates entry_block_mask (sqv_pair.cuh) for the
//      frame's entries, now sorted.
//
// One launch replaces the entry-count scan, emit, the two radix passes
// (histogram, scan, scatter each), the tile-bound search and the block-mask
// kernel.  Its few long-lived CTAs displace few evaluator CTAs while they run
// under the previous batch's evaluation; the replaced kernels were tens of
// thousands of short CTAs, each holding an evaluator slot.
#include "sqv_kernels.cuh"
#include "sqv_pair.cuh"

namespace sqv {

namespace {

constexpr int kBinThreads = 256;
constexpr int kBinWarps = kBinThreads / 32;

__global__ void __launch_bounds__(kBinThreads) bin_frames_kernel(BinArgs A) {
  extern __shared__ int sm[];
  __shared__ int s_red[kBinWarps];
  const int T = A.tiles_per_frame;
  int* cnt = sm;      // [T]: tile counts, then the tiles' offsets within the frame
  int* wc = sm + T;   // [8][T]: per-warp counts, then the warps' running ranks
  const int f = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N = A.n_prims;
  const int64_t fb = (int64_t)f * N;

  // frame base: the entries of the earlier frames (prep's per-frame counts)
  int part = 0;
  for (int j = tid; j < f; j += kBinThreads) part += A.frame_count[j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if (lane == 0) s_red[warp] = part;
  for (int i = tid; i < kBinWarps * T; i += kBinThreads) wc[i] = 0;
  __syncthreads();
  int base = 0;
#pragma unroll
  for (int w = 0; w < kBinWarps; ++w) base += s_red[w];

  // this warp's contiguous share of the frame's primitives
  const int per = (N + kBinWarps - 1) / kBinWarps;
  const int p0 = min(N, warp * per), p1 = min(N, p0 + per);
  int* my = wc + warp * T;
  auto rect = [&](int64_t gi, int& tx0, int& nxr, int& ty0, int& nyr, int& tz0) {
    const int* w = A.windows + 6 * gi;
    tx0 = w[0] / kTileX;
    ty0 = w[1] / kTileY;
    tz0 = w[2] / kTileZ;
    nxr = w[3] / kTileX - tx0 + 1;
    nyr = w[4] / kTileY - ty0 + 1;
  };

  // 1. counts per warp row
  for (int i = p0 + lane; i < p1; i += 32) {
    const int c = A.counts[fb + i];
    if (c == 0) continue;
    int tx0, nxr, ty0, nyr, tz0;
    rect(fb + i, tx0, nxr, ty0, nyr, tz0);
    for (int j = 0; j < c; ++j) {
      const int dx = j % nxr, r = j / nxr, dy = r % nyr, dz = r / nyr;
      atomicAdd(&my[(tx0 + dx) + A.ntx * ((ty0 + dy) + A.nty * (tz0 + dz))], 1);
    }
  }
  __syncthreads();
  // 2. per tile: the warps' first ranks and the tile's count
  for (int t = tid; t < T; t += kBinThreads) {
    int s = 0;
#pragma unroll
    for (int w = 0; w < kBinWarps; ++w) {
      const int v = wc[w * T + t];
      wc[w * T + t] = s;
      s += v;
    }
    cnt[t] = s;
  }
  __syncthreads();
  // exclusive scan of the tile counts: contiguous segments per thread
  const int seg = (T + kBinThreads - 1) / kBinThreads;
  const int t0 = min(T, tid * seg), t1 = min(T, t0 + seg);
  int loc = 0;
  for (int t = t0; t < t1; ++t) loc += cnt[t];
  int x = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();  // every thread has read its segment of cnt and s_red is free
  if (lane == 31) s_red[warp] = x;
  __syncthreads();
  int run = x - loc;
  for (int w = 0; w < warp; ++w) run += s_red[w];
  int total = 0;
#pragma unroll
  for (int w = 0; w < kBinWarps; ++w) total += s_red[w];
  const int64_t tg0 = (int64_t)f * T;
  for (int t = t0; t < t1; ++t) {
    const int v = cnt[t];
    cnt[t] = run;
    A.tile_off[tg0 + t] = base + run;
    if (A.deep_min >= 0 && v > A.deep_min) A.deep_tiles[atomicAdd(A.deep_count, 1)] = (int)(tg0 + t);
    run += v;
  }
  if (f == A.n_frames - 1 && tid == 0) A.tile_off[(int64_t)A.n_frames * T] = base + total;
  __syncthreads();

  // 3. ordered scatter: this warp's primitives in ascending id
  for (int i0 = p0; i0 < p1; i0 += 32) {
    const int i = i0 + lane;
    int c = 0, tx0 = 0, nxr = 1, ty0 = 0, nyr = 1, tz0 = 0;
    if (i < p1) {
      c = A.counts[fb + i];
      if (c) rect(fb + i, tx0, nxr, ty0, nyr, tz0);
    }
    const int kn = min(32, p1 - i0);
    for (int k = 0; k < kn; ++k) {
      const int ck = __shfl_sync(0xffffffffu, c, k);
      if (ck == 0) continue;
      const int bx = __shfl_sync(0xffffffffu, tx0, k), nx = __shfl_sync(0xffffffffu, nxr, k);
      const int by = __shfl_sync(0xffffffffu, ty0, k), ny = __shfl_sync(0xffffffffu, nyr, k);
      const int bz = __shfl_sync(0xffffffffu, tz0, k);
      for (int j = lane; j < ck; j += 32) {
        const int dx = j % nx, r = j / nx, dy = r % ny, dz = r / ny;
        const int t = (bx + dx) + A.ntx * ((by + dy) + A.nty * (bz + dz));
        const int pos = base + cnt[t] + my[t];
        my[t] += 1;  // distinct tiles within one primitive
        A.keys[pos] = (uint32_t)(tg0 + t);
        A.vals[pos] = i0 + k;
      }
      __syncwarp();  // this primitive's ranks before the next one's
    }
  }

  // 4. the block masks of the frame's (now sorted) entries
  if (A.bmask) {
    __syncthreads();  // the CTA's keys/vals writes are visible to the CTA
    for (int e = tid; e < total; e += kBinThreads) {
      const int pos = base + e;
      const int t = (int)(A.keys[pos] - (uint32_t)tg0);
      const int64_t g = fb + A.vals[pos];
      const int e_tile = (t + 1 < T ? cnt[t + 1] : total) - cnt[t];
      A.bmask[pos] = entry_block_mask(A.recs + g * kRecWords,
                                      __ldg(A.lrows + g * A.lrow + (A.lrow - 1)), e_tile,
                                      t % A.ntx, (t / A.ntx) % A.nty, t / (A.ntx * A.nty),
                                      A.acc_c);
    }
  }
}

}  // namespace

size_t bin_frames_smem(int tiles_per_frame) {
  return (size_t)(kBinWarps + 1) * (size_t)tiles_per_frame * sizeof(int);
}

bool bin_frames_supported(int tiles_per_frame) {
  return bin_frames_smem(tiles_per_frame) <= 200 * 1024;
}

int bin_frames_launch(const BinArgs& A, cudaStream_t s) {
  if (A.n_frames <= 0) return SQV_OK;
  const size_t smem = bin_frames_smem(A.tiles_per_frame);
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(bin_frames_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess)
    return check_launch("bin_frames_kernel attribute");
  bin_frames_kernel<<<A.n_frames, kBinThreads, smem, s>>>(A);
  count_launch();
  return check_launch("bin_frames_kernel");
}

}  // namespace sqv
