// Latency probe: dependent chains of FFMA, FFMA2, MUFU.EX2, MUFU.LG2 (one
// warp, clock64 around N dependent ops).  Dev tool, not part of the build.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(float* out, long long* cyc, float s) {
  float a = s, b = s * 0.5f;
  float2 p = make_float2(s, s * 0.25f), q = make_float2(1.0000001f, 0.9999999f);
  long long t0, t1;
  const int N = 1024;
  // FFMA chain
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) a = fmaf(a, 1.0000001f, b);
  t1 = clock64();
  cyc[0] = t1 - t0;
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) p = __ffma2_rn(p, q, p);
  t1 = clock64();
  cyc[1] = t1 - t0;
  float e = s;
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(e));
  t1 = clock64();
  cyc[2] = t1 - t0;
  float l = s + 2.0f;
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) asm volatile("lg2.approx.ftz.f32 %0, %0;" : "+f"(l));
  t1 = clock64();
  cyc[3] = t1 - t0;
  float2 m = make_float2(s, s);
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) m = __fmul2_rn(m, q);
  t1 = clock64();
  cyc[4] = t1 - t0;
  out[threadIdx.x] = a + p.x + p.y + e + l + m.x;
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 128); cudaMalloc(&c, 64);
  k<<<1, 32>>>(o, c, 0.5f);
  long long h[5]; cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
  const char* nm[5] = {"FFMA", "FFMA2", "MUFU.EX2", "MUFU.LG2", "FMUL2"};
  for (int i = 0; i < 5; ++i) printf("%-9s dependent latency %.2f cycles\n", nm[i], h[i] / 1024.0);
  return 0;
}
