// pk_umma.cuh — minimal sm_100a tcgen05 (UMMA) / TMEM / mbarrier layer.
//
// Written against the PTX ISA for tcgen05 (CUDA 12.9); descriptor bit
// layouts follow the sm_100 UMMA shared-memory and instruction descriptors.
// Only what the pack kernels use:
//   * kind::tf32 MMAs, cta_group::1, M = 128, fp32 accumulators in TMEM,
//     operands in shared memory in the SWIZZLE_NONE canonical layouts;
//   * 3xTF32: a = a_hi + a_lo (a_hi = rna_tf32(a), a_lo = a - a_hi), so
//     A·B ≈ A_hi·B_hi + A_hi·B_lo + A_lo·B_hi accumulates in fp32 to ~2^-21
//     relative — the fp32 parity contract (rel 1e-4) that plain TF32 misses;
//   * TMEM alloc / dealloc, 32x32b loads for the epilogue.
//
// Shared-memory operand layouts (SWIZZLE_NONE, 16-byte core-matrix rows):
//   K-major  (k contiguous):   elem(r, k) at ((k/4)·ROWS + r)·16 + (k%4)·4 bytes
//                              → core matrix = 8 rows × 16 B; SBO = 128 B
//                                (next 8 rows), LBO = ROWS·16 B (next 4 k).
//                                One K-step (8 tf32) starts at base + s·2·ROWS·16.
// (Only K-major is used: staging passes transpose while splitting hi/lo;
// verified on B200 by tools/umma_selftest.cu.)
#pragma once
#include <cstdint>

namespace umma {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- descriptors ------------------------------------------------------------
// shared-memory matrix descriptor, SWIZZLE_NONE, version 1 (sm_100)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version = 1
  // base_offset = 0, lbo_mode = 0, layout_type (bits 61-63) = 0 = SWIZZLE_NONE
  return d;
}

// instruction descriptor: kind::tf32, fp32 accumulate, dense
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4)                     // c_format = F32
         | (2u << 7)                   // a_format = TF32
         | (2u << 10)                  // b_format = TF32
         | ((a_mn ? 1u : 0u) << 15)    // a_major
         | ((b_mn ? 1u : 0u) << 16)    // b_major
         | ((uint32_t)(N >> 3) << 17)  // n_dim
         | ((uint32_t)(M >> 4) << 24); // m_dim
}

// byte offsets of the canonical layouts (see header)
__host__ __device__ constexpr uint32_t kmaj_off(int r, int k, int rows) {
  return (uint32_t)(((k >> 2) * rows + r) * 16 + (k & 3) * 4);
}
// descriptor of K-step s (8 tf32 along k) of an operand with `rows` rows
__device__ __forceinline__ uint64_t kmaj_desc(uint32_t base, int rows, int s) {
  return sdesc(base + (uint32_t)(s * 2 * rows * 16), (uint32_t)(rows * 16), 128u);
}

// ---- tf32 split -------------------------------------------------------------
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ void split3(float x, float& hi, float& lo) {
  hi = tf32_rna(x);
  lo = tf32_rna(x - hi);
}

// ---- MMA --------------------------------------------------------------------
// D[tmem] (+)= A[smem] · B[smem]ᵀ   (A: M×K, B: N×K, 8-deep K for tf32)
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, bool accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
      :
      : "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"((uint32_t)accumulate));
}

// all prior tcgen05.mma of this thread arrive on `mbar` when complete
__device__ __forceinline__ void commit(uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               :
               : "r"(smem_u32(mbar))
               : "memory");
}

__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// generic-proxy smem writes → visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---- mbarrier ----------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(mbar)),
      "r"(parity)
      : "memory");
}

// ---- cluster barrier ----------------------------------------------------------
__device__ __forceinline__ void cluster_sync() {  // arrive.release + wait.acquire
  asm volatile("barrier.cluster.arrive.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}

// ---- distributed shared memory ---------------------------------------------
// load the float at local shared address `la` of cluster CTA `rank`
__device__ __forceinline__ float dsmem_ld(uint32_t la, uint32_t rank) {
  uint32_t ra;
  float v;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(rank));
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(ra));
  return v;
}

// the 16-byte vector at local shared address `la` (16-B aligned) of cluster CTA
// `rank`: one DSMEM transaction for four consecutive floats
__device__ __forceinline__ float4 dsmem_ld4(uint32_t la, uint32_t rank) {
  uint32_t ra;
  float4 v;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(rank));
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(ra));
  return v;
}

// ---- mbarrier transaction counts (TMA loads complete on them) ----------------
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)),
               "r"(bytes)
               : "memory");
}

// ---- TMEM ----------------------------------------------------------------------
// one full warp calls alloc/dealloc; `ncols` power of two >= 32
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
// warp w (w%4 = lane quarter) loads lane (32·(w%4) + laneid), columns col..col+7
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__host__ __device__ constexpr uint32_t tmem_cols_pow2(uint32_t n) {
  return n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : n <= 256 ? 256 : 512;
}

}  // namespace umma
