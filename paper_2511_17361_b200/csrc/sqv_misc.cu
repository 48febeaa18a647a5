// sqv_misc.cu — finalize (tau sweeps), K6 confusion counts, point density.
#include "sqv_kernels.cuh"

namespace sqv {

namespace {

// finalize: one thread per voxel.
__global__ void finalize_kernel(const float* __restrict__ v_o, const float* __restrict__ v_c,
                                int64_t n, int C, float tau, int free_label,
                                uint8_t* __restrict__ labels) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    uint8_t lab;
    if (v_o[v] < tau) {
      lab = (uint8_t)free_label;
    } else {
      const float* c = v_c + v * C;
      int best = 0;
      float bv = c[0];
      for (int k = 1; k < C; ++k)
        if (c[k] > bv) {
          bv = c[k];
          best = k;
        }
      lab = (uint8_t)best;
    }
    labels[v] = lab;
  }
}

// K6: (C+1)^2 confusion counts, row = gt, col = pred, label >= C -> C (free).
// Shared-memory int32 histogram per CTA (16-byte vector loads), flushed with
// 64-bit atomics; integer sums are exact, so the result is deterministic.
constexpr int kCmThreads = 512;
__global__ void __launch_bounds__(kCmThreads) confusion_kernel(const uint8_t* __restrict__ pred,
                                                               const uint8_t* __restrict__ gt,
                                                               int64_t n, int C,
                                                               unsigned long long* cm) {
  extern __shared__ int h[];
  const int K = C + 1;
  for (int k = threadIdx.x; k < K * K; k += blockDim.x) h[k] = 0;
  __syncthreads();
  const int64_t n16 = n / 16;
  const uint4* p4 = reinterpret_cast<const uint4*>(pred);
  const uint4* g4 = reinterpret_cast<const uint4*>(gt);
  const bool aligned = ((reinterpret_cast<uintptr_t>(pred) | reinterpret_cast<uintptr_t>(gt)) & 15) == 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t done = 0;
  if (aligned) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) {
      const uint4 a = p4[i], b = g4[i];
      const uint32_t pa[4] = {a.x, a.y, a.z, a.w}, gb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int w = 0; w < 4; ++w)
#pragma unroll
        for (int byte = 0; byte < 4; ++byte) {
          const int p = min((int)((pa[w] >> (8 * byte)) & 255u), C);
          const int g = min((int)((gb[w] >> (8 * byte)) & 255u), C);
          atomicAdd(&h[g * K + p], 1);
        }
    }
    done = n16 * 16;
  }
  for (int64_t i = done + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int p = min((int)pred[i], C), g = min((int)gt[i], C);
    atomicAdd(&h[g * K + p], 1);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < K * K; k += blockDim.x)
    if (h[k]) atomicAdd(cm + k, (unsigned long long)h[k]);
}

// density / inside-outside at arbitrary world points (core.py:237-282):
// FP64 setup + FP64 transform, FP32 field on the SFU (same field_F7 as the
// evaluator).
__global__ void density_kernel(sqv_prims P, const double* __restrict__ points,
                               const int32_t* __restrict__ pair_prim, int64_t n,
                               float* __restrict__ Fout, float* __restrict__ dout) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int j = pair_prim[k];
  const PrimF64 Q = prim_setup(P.mu + 3 * j, P.scale + 3 * j, P.rot + 4 * j, P.opacity[j],
                               P.eps + 2 * j, P.logits + (int64_t)P.n_classes * j, P.n_classes);
  if (Q.bad) {
    Fout[k] = __int_as_float(0x7fc00000);
    dout[k] = __int_as_float(0x7fc00000);
    return;
  }
  const double d0 = points[3 * k] - Q.mu[0], d1 = points[3 * k + 1] - Q.mu[1],
               d2 = points[3 * k + 2] - Q.mu[2];
  const float x0 = (float)(Q.M[0] * d0 + Q.M[1] * d1 + Q.M[2] * d2);
  const float x1 = (float)(Q.M[3] * d0 + Q.M[4] * d1 + Q.M[5] * d2);
  const float x2 = (float)(Q.M[6] * d0 + Q.M[7] * d1 + Q.M[8] * d2);
  const float F = field_F6(x0, x1, x2, (float)(2.0 / Q.e2), (float)(Q.e2 / Q.e1),
                          (float)(2.0 / Q.e1));
  Fout[k] = fminf(F, kFCap);
  dout[k] = density_of(F);
}

// Pipe microbenchmarks: 8 independent chains per thread so the pipe, not
// latency, is the limit; grid = 8 CTAs x 256 threads per SM.
constexpr int kMbIters = 4096;
__global__ void __launch_bounds__(256) mb_mufu_kernel(float* sink, float seed) {
  float v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = seed + 0.01f * (threadIdx.x + k);
  for (int it = 0; it < kMbIters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = (k & 1) ? lg2(v[k]) : ex2(v[k]);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += v[k];
  if (s == 1234.5f) sink[threadIdx.x] = s;
}
__global__ void __launch_bounds__(256) mb_ffma_kernel(float* sink, float seed) {
  float v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = seed + 0.01f * (threadIdx.x + k);
  for (int it = 0; it < kMbIters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = fmaf(v[k], 0.999f, 0.0001f);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += v[k];
  if (s == 1234.5f) sink[threadIdx.x] = s;
}

}  // namespace

int microbench(int which, double* ops_per_s, cudaStream_t s) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = sms * 8;
  float* sink = nullptr;
  if (cudaMallocAsync(&sink, 256 * sizeof(float), s) != cudaSuccess)
    return check_launch("microbench alloc");
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best = 0.0;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0, s);
    if (which == 0)
      mb_mufu_kernel<<<blocks, 256, 0, s>>>(sink, 1.5f);
    else
      mb_ffma_kernel<<<blocks, 256, 0, s>>>(sink, 1.5f);
    count_launch();
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)blocks * 256 * kMbIters * 8;
    if (rep > 0 && ms > 0) best = fmax(best, ops / (ms * 1e-3));
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFreeAsync(sink, s);
  *ops_per_s = best;
  return check_launch("microbench");
}

int finalize_launch(const float* v_o, const float* v_c, int64_t n, int C, float tau,
                    int free_label, uint8_t* labels, cudaStream_t s) {
  if (n <= 0) return SQV_OK;
  const int64_t nb = (n + 255) / 256;
  finalize_kernel<<<(int)(nb < 148 * 64 ? nb : 148 * 64), 256, 0, s>>>(v_o, v_c, n, C, tau,
                                                                       free_label, labels);
  count_launch();
  return check_launch("finalize_kernel");
}

int confusion_launch(const uint8_t* pred, const uint8_t* gt, int64_t n, int C, int64_t* cm,
                     cudaStream_t s) {
  if (n <= 0) return SQV_OK;
  const int K = C + 1;
  const int smem = K * K * 4;
  int64_t nb = (n / 16 + kCmThreads - 1) / kCmThreads;
  if (nb > 148 * 4) nb = 148 * 4;
  if (nb < 1) nb = 1;
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(confusion_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
          cudaSuccess)
    return check_launch("confusion attribute");
  confusion_kernel<<<(int)nb, kCmThreads, smem, s>>>(pred, gt, n, C,
                                                     reinterpret_cast<unsigned long long*>(cm));
  count_launch();
  return check_launch("confusion_kernel");
}

int density_launch(const sqv_prims* P, const double* points, const int32_t* pair_prim, int64_t n,
                   float* F, float* density, cudaStream_t s) {
  if (n <= 0) return SQV_OK;
  density_kernel<<<(int)((n + 255) / 256), 256, 0, s>>>(*P, points, pair_prim, n, F, density);
  count_launch();
  return check_launch("density_kernel");
}

}  // namespace sqv
