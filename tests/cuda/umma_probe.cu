// umma_probe.cu — standalone GPU probe of the tcgen05 kind::tf32 operand
// layouts (one CTA, one M=128 N=32 K=8 MMA, result read back with
// tcgen05.ld and compared with a host GEMM).  Used to pin the layout that
// sqv_eval_tc.cu relies on; prints one line per layout combination.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o umma_probe umma_probe.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "../../paper_2511_17361_b200/csrc/sqv_tc.cuh"

using namespace sqv;

// layout ids
//  0: K-major, SWIZZLE_32B   (rows of 32 B = 8 tf32; 8-row atoms of 256 B; SBO = 256)
//  1: MN-major, SWIZZLE_128B (rows of 128 B = 32 mn; 8 k-rows per 1 KB atom; LBO = 1024)
//  2: MN-major, SWIZZLE_NONE (core matrix 4 mn x 8 k = 128 B; SBO = 128 along mn)
//  3: K-major, SWIZZLE_NONE  (core matrix 8 mn x 4 k = 128 B; LBO = k-chunk stride, SBO = 128)
//  4: MN-major, SWIZZLE_128B_BASE32B (rows of 128 B = 32 mn, 4 k-rows per 512 B atom,
//     32-byte chunks XOR row; LBO = mn-atom stride 512, SBO = k-group stride)
struct Lay {
  int id;
  uint32_t lbo, sbo;
  uint32_t type;  // descriptor layout type
  int major;      // 0 K, 1 MN
};

__device__ uint32_t off_of(int id, int mn, int k, int mn_extent) {
  switch (id) {
    case 0: return (uint32_t)((mn >> 3) * 256 + (mn & 7) * 32 + ((((k >> 2) ^ ((mn >> 2) & 1))) << 4) + ((k & 3) << 2));
    case 1: return (uint32_t)((mn >> 5) * 1024 + k * 128 + ((((mn >> 2) & 7) ^ k) << 4) + ((mn & 3) << 2));
    case 2: return (uint32_t)((mn >> 2) * 128 + k * 16 + ((mn & 3) << 2));
    case 3: return tc::kmajor_chunk(mn, k >> 2, mn_extent) + ((k & 3) << 2);
    default:
      return (uint32_t)((k >> 2) * (mn_extent / 32) * 512 + (mn >> 5) * 512 + (k & 3) * 128 +
                        ((((mn >> 3) & 3) ^ (k & 3)) << 5) + ((mn & 7) << 2));
  }
}

__device__ uint64_t desc_of(uint32_t saddr, Lay L) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((L.lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((L.sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | ((uint64_t)L.type << 61);
}

__global__ void probe(const float* A, const float* B, float* D, Lay la, Lay lb) {
  extern __shared__ __align__(16) uint8_t raw[];
  uint8_t* smem = raw + ((1024 - (tc::smem_u32(raw) & 1023)) & 1023);
  uint8_t* sa = smem;          // 16 KB
  uint8_t* sb = smem + 16384;  // 4 KB
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 20480);
  uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + 20488);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 20480; i += blockDim.x) smem[i] = 0;
  __syncthreads();
  for (int i = tid; i < 128 * 8; i += blockDim.x) {
    const int m = i / 8, k = i % 8;
    *reinterpret_cast<float*>(sa + off_of(la.id, m, k, 128)) = A[m * 8 + k];
  }
  for (int i = tid; i < 8 * 32; i += blockDim.x) {
    const int k = i / 32, n = i % 32;
    *reinterpret_cast<float*>(sb + off_of(lb.id, n, k, 32)) = B[k * 32 + n];
  }
  if (warp == 0) {
    tc::tmem_alloc(tptr, 32);
    tc::tmem_relinquish();
  }
  if (tid == 0) {
    tc::mbar_init(bar, 1);
    tc::fence_mbar_init();
  }
  tc::fence_proxy_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = *tptr;
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)la.major << 15) |
                           ((uint32_t)lb.major << 16) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
    tc::mma_tf32(tbase, desc_of(tc::smem_u32(sa), la), desc_of(tc::smem_u32(sb), lb), idesc, 0u);
    tc::mma_commit(bar);
  }
  __syncwarp();
  tc::mbar_wait(bar, 0);
  tc::fence_after_sync();
  float vals[32];
  tc::tmem_ld_32x32b_x32(tbase + ((uint32_t)(warp * 32) << 16), vals);
  for (int n = 0; n < 32; ++n) D[(warp * 32 + lane) * 32 + n] = vals[n];
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tbase, 32);
  }
}

int main() {
  static float hA[128 * 8], hB[8 * 32], ref[128 * 32], hD[128 * 32];
  for (int i = 0; i < 128 * 8; ++i) hA[i] = (float)((i * 7) % 13) - 6.0f;
  for (int i = 0; i < 8 * 32; ++i) hB[i] = (float)((i * 5) % 11) - 5.0f;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 32; ++n) {
      float s = 0;
      for (int k = 0; k < 8; ++k) s += hA[m * 8 + k] * hB[k * 32 + n];
      ref[m * 32 + n] = s;
    }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, sizeof hA);
  cudaMalloc(&dB, sizeof hB);
  cudaMalloc(&dD, sizeof hD);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 24576);
  // A candidates (mn extent 128) and B candidates (mn extent 32)
  // MN-major tf32 works only with SWIZZLE_128B_BASE32B (layout 4); the
  // MN-major SWIZZLE_NONE / SWIZZLE_128B encodings read zeros (probed).
  const Lay As[] = {{0, 16, 256, 6, 0}, {3, 2048, 128, 0, 0}, {4, 512, 2048, 1, 1}};
  const Lay Bs[] = {{0, 16, 256, 6, 0}, {3, 512, 128, 0, 0}, {4, 512, 512, 1, 1}};
  int failures = 0;
  for (const Lay& la : As)
    for (const Lay& lb : Bs) {
      cudaMemset(dD, 0, sizeof hD);
      probe<<<1, 128, 24576>>>(dA, dB, dD, la, lb);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("A%d(lbo %u sbo %u) B%d: CUDA error %s\n", la.id, la.lbo, la.sbo, lb.id,
               cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
      double err = 0;
      int bad = 0;
      for (int i = 0; i < 128 * 32; ++i) {
        const double d = fabs(hD[i] - ref[i]);
        err = fmax(err, d);
        bad += d > 0.5;
      }
      printf("A%d lbo=%-5u sbo=%-5u | B%d lbo=%-5u sbo=%-5u : bad %4d  max|err| %g %s\n", la.id,
             la.lbo, la.sbo, lb.id, lb.lbo, lb.sbo, bad, err, bad == 0 ? "  <== OK" : "");
      failures += bad != 0;
    }
  return failures ? 2 : 0;
}
