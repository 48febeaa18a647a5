// sqv_sort.cu — K2 device-wide exclusive prefix scan and K4 stable LSD radix
// sort, hand-written (no CUB).  Used for: per-primitive bin offsets, per-tile
// list offsets and the radix digit histograms.  Both are deterministic: the
// bins they produce are bit-identical to the oracle's (tests/test_gpu_*).
#include "sqv_kernels.cuh"

namespace sqv {

namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;
constexpr int kSpineThreads = 1024;

constexpr int kRadixThreads = 256;
constexpr int kRadixRounds = 8;
constexpr int kRadixTile = kRadixThreads * kRadixRounds;
constexpr int kRadixWarps = kRadixThreads / 32;

// Block-wide exclusive scan of one int per thread; returns the exclusive
// prefix and sets *total.  `sh` needs 32 ints.
template <int NT>
__device__ __forceinline__ int block_excl_scan(int v, int* sh, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int s = lane < NT / 32 ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    sh[lane] = s;  // inclusive warp-total prefix
  }
  __syncthreads();
  const int before = warp > 0 ? sh[warp - 1] : 0;
  *total = sh[NT / 32 - 1];
  __syncthreads();
  return before + x - v;
}

__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(const int* __restrict__ in,
                                                                   int64_t n, int* tmp) {
  __shared__ int sh[32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k)
    if (base + k < n) s += in[base + k];
  int total;
  block_excl_scan<kScanThreads>(s, sh, &total);
  if (threadIdx.x == 0) tmp[blockIdx.x] = total;
}

// Single block: exclusive scan of the nb block sums in place, total -> out[n].
__global__ void __launch_bounds__(kSpineThreads) scan_spine_kernel(int* tmp, int nb, int* out,
                                                                   int64_t n,
                                                                   long long* total64) {
  __shared__ int sh[32];
  int carry = 0;
  for (int b0 = 0; b0 < nb; b0 += kSpineThreads) {
    const int b = b0 + threadIdx.x;
    const int v = b < nb ? tmp[b] : 0;
    int total;
    const int ex = block_excl_scan<kSpineThreads>(v, sh, &total);
    if (b < nb) tmp[b] = carry + ex;
    carry += total;
  }
  if (threadIdx.x == 0) {
    out[n] = carry;
    if (total64) *total64 = carry;
  }
}

__global__ void __launch_bounds__(kScanThreads) scan_final_kernel(const int* __restrict__ in,
                                                                  int* __restrict__ out,
                                                                  int64_t n,
                                                                  const int* __restrict__ tmp) {
  __shared__ int sh[32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int v[kScanItems];
  int s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = base + k < n ? in[base + k] : 0;
    s += v[k];
  }
  int total;
  int run = block_excl_scan<kScanThreads>(s, sh, &total) + tmp[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k < n) out[base + k] = run;
    run += v[k];
  }
}

// ---- radix sort -------------------------------------------------------------

__global__ void __launch_bounds__(kRadixThreads) radix_hist_kernel(const uint32_t* __restrict__ keys,
                                                                   int64_t n, int shift, int nb,
                                                                   int* __restrict__ hist) {
  __shared__ int h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kRadixTile;
#pragma unroll
  for (int r = 0; r < kRadixRounds; ++r) {
    const int64_t idx = base + r * kRadixThreads + threadIdx.x;
    if (idx < n) atomicAdd(&h[(keys[idx] >> shift) & 255u], 1);
  }
  __syncthreads();
  hist[(int64_t)threadIdx.x * nb + blockIdx.x] = h[threadIdx.x];
}

// Stable scatter: keys are ranked in their original order within the block
// (rounds in order, warps in order within a round, lanes in order within a
// warp via match_any + lanemask), and blocks are ordered by the digit-major
// scan of the histograms.
__global__ void __launch_bounds__(kRadixThreads) radix_scatter_kernel(
    const uint32_t* __restrict__ kin, const int* __restrict__ vin, uint32_t* __restrict__ kout,
    int* __restrict__ vout, int64_t n, int shift, int nb, const int* __restrict__ hist_off) {
  __shared__ int run[256];
  __shared__ int wcnt[kRadixWarps][256];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  run[tid] = hist_off[(int64_t)tid * nb + blockIdx.x];
#pragma unroll
  for (int w = 0; w < kRadixWarps; ++w) wcnt[w][tid] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kRadixTile;
  const unsigned lt = (1u << lane) - 1u;
  for (int r = 0; r < kRadixRounds; ++r) {
    const int64_t idx = base + r * kRadixThreads + tid;
    const bool valid = idx < n;
    uint32_t key = 0;
    int val = 0;
    int d = 256;
    if (valid) {
      key = kin[idx];
      val = vin[idx];
      d = (int)((key >> shift) & 255u);
    }
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const int rank = __popc(peers & lt);
    if (valid && rank == 0) wcnt[warp][d] = __popc(peers);
    __syncthreads();
    if (valid) {
      int pos = run[d] + rank;
      for (int w = 0; w < warp; ++w) pos += wcnt[w][d];
      kout[pos] = key;
      vout[pos] = val;
    }
    __syncthreads();
    int add = 0;
#pragma unroll
    for (int w = 0; w < kRadixWarps; ++w) {
      add += wcnt[w][tid];
      wcnt[w][tid] = 0;
    }
    run[tid] += add;
    __syncthreads();
  }
}

}  // namespace

int64_t scan_tmp_ints(int64_t n) { return (n + kScanTile - 1) / kScanTile + 1; }

int scan_exclusive(const int* in, int* out, int64_t n, int* tmp, long long* total64,
                   cudaStream_t s) {
  const int nb = (int)((n + kScanTile - 1) / kScanTile);
  if (nb > 0) {
    scan_reduce_kernel<<<nb, kScanThreads, 0, s>>>(in, n, tmp);
    count_launch();
  }
  scan_spine_kernel<<<1, kSpineThreads, 0, s>>>(tmp, nb, out, n, total64);
  count_launch();
  if (nb > 0) {
    scan_final_kernel<<<nb, kScanThreads, 0, s>>>(in, out, n, tmp);
    count_launch();
  }
  return check_launch("scan_exclusive");
}

int64_t radix_tmp_ints(int64_t n) {
  const int64_t nb = (n + kRadixTile - 1) / kRadixTile;
  const int64_t h = 256 * nb;
  return 2 * (h + 1) + scan_tmp_ints(h);
}

int radix_sort(uint32_t* keys, int* vals, uint32_t* keys_alt, int* vals_alt, int64_t n, int bits,
               int* tmp, int* which, cudaStream_t s) {
  *which = 0;
  if (n <= 0 || bits <= 0) return SQV_OK;
  const int nb = (int)((n + kRadixTile - 1) / kRadixTile);
  const int64_t h = 256LL * nb;
  int* hist = tmp;
  int* hist_off = tmp + (h + 1);
  int* stmp = tmp + 2 * (h + 1);
  uint32_t* kin = keys;
  int* vin = vals;
  uint32_t* kout = keys_alt;
  int* vout = vals_alt;
  for (int shift = 0; shift < bits; shift += 8) {
    radix_hist_kernel<<<nb, kRadixThreads, 0, s>>>(kin, n, shift, nb, hist);
    count_launch();
    int rc = scan_exclusive(hist, hist_off, h, stmp, nullptr, s);
    if (rc) return rc;
    radix_scatter_kernel<<<nb, kRadixThreads, 0, s>>>(kin, vin, kout, vout, n, shift, nb,
                                                      hist_off);
    count_launch();
    rc = check_launch("radix_scatter");
    if (rc) return rc;
    uint32_t* tk = kin;
    kin = kout;
    kout = tk;
    int* tv = vin;
    vin = vout;
    vout = tv;
    *which ^= 1;
  }
  return SQV_OK;
}

}  // namespace sqv
