// sqv_tc.cuh — thin inline-PTX helpers for tcgen05 (TMEM, UMMA), mbarriers
// and async-proxy fences, sm_100a.
#pragma once

#include <stdint.h>

namespace sqv {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- cp.async (global -> shared, no register round trip) ----------------
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
// wait until at most N of this thread's committed groups are pending
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---- bulk async copy shared -> global (epilogue rows) --------------------
__device__ __forceinline__ void bulk_store(void* gdst, uint32_t ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(ssrc), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit_wait_read() {
  asm volatile("cp.async.bulk.commit_group;\n\tcp.async.bulk.wait_group.read 0;" ::: "memory");
}

// ---- TMEM ---------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst)),
               "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tmem_relinquish() {
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void fence_before_sync() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after_sync() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// generic-proxy smem stores -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// 32 lanes x 32 consecutive 32-bit columns -> 32 registers per thread.
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 lanes x the first 20 columns (x16 + x4): enough for 18 classes + sigma,
// 5/8 of the x32 load's TMEM read traffic.  v[20..31] are left untouched.
__device__ __forceinline__ void tmem_ld_32x32b_x20(uint32_t taddr, float (&v)[32]) {
  uint32_t r[20];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19])
               : "r"(taddr + 16u));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 20; ++i) v[i] = __uint_as_float(r[i]);
}

// ---- mbarrier ---------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// ---- UMMA -------------------------------------------------------------------
// D[tmem] (+)= A[smem] * B[smem], kind::tf32, cta_group::1.
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on `bar` when all prior tcgen05 ops of this thread complete
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// One K step of the 3xTF32 split (hi*hi + hi*lo + lo*hi) and its commit,
// issued by one elected lane of the calling (converged) warp: elect.sync
// inside the asm, so ptxas needs no per-instruction elect loop.  `first`
// = 1 starts the accumulator (enable-input-d off for the first MMA).
__device__ __forceinline__ void mma3_tf32_commit(uint32_t d_tmem, uint64_t a_hi, uint64_t a_lo,
                                                 uint64_t b_hi, uint64_t b_lo, uint32_t idesc,
                                                 uint32_t first, uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e, acc;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.eq.b32 acc, %6, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %3, %5, acc;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %4, %5, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %2, %3, %5, 1;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%7];\n}" ::"r"(
          d_tmem),
      "l"(a_hi), "l"(a_lo), "l"(b_hi), "l"(b_lo), "r"(idesc), "r"(first), "r"(smem_u32(bar))
      : "memory");
}

// Instruction descriptor: D f32, A/B tf32, M x N; a_mn/b_mn select
// MN-major operands (bits 15/16).
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int a_mn, int b_mn) {
  return (1u << 4)                  // D format f32
         | (2u << 7)                // A format tf32
         | (2u << 10)               // B format tf32
         | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

// MN-major 32-bit operands need the SWIZZLE_128B_BASE32B mode (layout type
// 1; every other MN-major encoding reads zeros for tf32 — pinned by
// tests/cuda/umma_probe.cu).  Canonical form: 128-byte rows of 32 mn
// elements, 4 k-rows per 512-byte atom, the four 32-byte chunks of a row
// XOR-ed with the row index; LBO = stride between mn atoms, SBO = stride
// between groups of 4 k.
__device__ __forceinline__ uint64_t smem_desc_mn32(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (1ull << 61);
}

// Byte offset of element (mn, k) in such an operand with `mn_extent` rows
// (mn atoms 512 B apart, k groups mn_extent*16 B apart).  Elements mn..mn+3
// (mn % 4 == 0) are 16 contiguous bytes.
__device__ __forceinline__ uint32_t mn32_offset(int mn, int k, int mn_extent) {
  return (uint32_t)((k >> 2) * mn_extent * 16 + (mn >> 5) * 512 + (k & 3) * 128 +
                    ((((mn >> 3) & 3) ^ (k & 3)) << 5) + ((mn & 7) << 2));
}

// Shared-memory matrix descriptor, SWIZZLE_NONE ("interleaved"), sm_100
// (version 1).  K-major canonical form (16-byte units):
//   ((8,m),2):((1,SBO),LBO) — core matrices of 8 rows x 16 B (4 tf32),
//   SBO = byte stride between 8-row groups, LBO = byte stride between the
//   two 16-byte K chunks of a K = 8 step.
__device__ __forceinline__ uint64_t smem_desc_kmajor(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

// Byte offset of the 16-byte chunk (row r, k in [4c, 4c+4)) of a K-major
// interleaved operand with `rows` rows: core matrices contiguous along rows
// (SBO = 128), the K chunks `rows * 16` bytes apart (LBO).
__device__ __forceinline__ uint32_t kmajor_chunk(int r, int c, int rows) {
  return (uint32_t)(c * rows * 16 + (r >> 3) * 128 + (r & 7) * 16);
}

}  // namespace tc
}  // namespace sqv
