// pk_tc.cuh — bf16 tcgen05 / TMA / cp.async layer for the conv pack path.
//
// Complements pk_umma.cuh (kind::tf32, SWIZZLE_NONE) with what the implicit-
// GEMM conv kernels need:
//   * kind::f16 (bf16 operands, fp32 accumulators in TMEM), cta_group::1;
//   * 128-byte-swizzled shared-memory operands, both majors:
//       K-major  : row r (an M or N index) holds 64 bf16 of K in 128 B; rows
//                  at 128 B, 8-row groups at SBO = 1024 B.  The 16-B chunk j
//                  of row r sits at chunk (j ^ (r & 7)) — the layout TMA
//                  writes with CU_TENSOR_MAP_SWIZZLE_128B for a {64, rows}
//                  box.  One UMMA K-step (16 bf16) advances the start address
//                  by 32 B inside the swizzle atom.
//       MN-major : row k (a K index) holds 64 bf16 of M (or N) in 128 B;
//                  8-k groups at SBO = 1024 B, 64-wide MN atoms at
//                  LBO = 64 rows · 128 B = 8192 B.  One K-step = 2 groups
//                  = +2048 B.
//   * TMA 2-D tile loads (cp.async.bulk.tensor) completing on an mbarrier;
//   * cp.async 16-B copies with zero fill (the im2col gathers).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>

#include "pk_umma.cuh"

namespace tc {

using umma::smem_u32;

// sm_100 shared-memory descriptor, SWIZZLE_128B (layout_type 2), version 1
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr, uint32_t lbo_bytes,
                                                uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

// SWIZZLE_32B (layout_type 6): 32-byte rows (16 bf16), 8-row atoms of 256 B.
//   K-major : one atom column = 16 K; an MMA K-step (16) is one whole slab of
//             rows x 32 B, so only SBO (8-row groups, 256 B) matters.
//   MN-major: atoms of 16 MN x 8 K; LBO = stride between 16-wide MN atoms,
//             SBO = stride between 8-row K groups (256 B).
__device__ __forceinline__ uint64_t sdesc_sw32(uint32_t saddr, uint32_t lbo_bytes,
                                               uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version
  d |= (uint64_t)6 << 61;  // SWIZZLE_32B
  return d;
}

// SWIZZLE_64B (layout_type 4), K-major: 64-byte rows (32 bf16 of K), 8-row atoms of
// 512 B (SBO); an MMA K-step (16) advances the start by 32 B inside the row
__device__ __forceinline__ uint64_t sdesc_sw64(uint32_t saddr, uint32_t lbo_bytes,
                                               uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version
  d |= (uint64_t)4 << 61;  // SWIZZLE_64B
  return d;
}

// instruction descriptor: kind::f16 with bf16 A/B, fp32 accumulate, dense
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4)                     // c_format = F32
         | (1u << 7)                   // a_format = BF16
         | (1u << 10)                  // b_format = BF16
         | ((a_mn ? 1u : 0u) << 15)    // a_major
         | ((b_mn ? 1u : 0u) << 16)    // b_major
         | ((uint32_t)(N >> 3) << 17)  // n_dim
         | ((uint32_t)(M >> 4) << 24); // m_dim
}

// byte offset of (row, 16-B chunk) in a K-major SW128 operand (64 bf16 / row)
__device__ __forceinline__ uint32_t kmaj_sw128(int row, int chunk) {
  return (uint32_t)((row >> 3) * 1024 + (row & 7) * 128 + ((chunk ^ (row & 7)) << 4));
}
// byte offset of (k row, 16-B chunk along MN) in an MN-major SW128 operand
// with 64 k rows per stage: 64-wide MN atoms are 8 KB apart
__device__ __forceinline__ uint32_t mnmaj_sw128(int k, int mn_chunk) {
  return (uint32_t)((mn_chunk >> 3) * 8192 + (k >> 3) * 1024 + (k & 7) * 128 +
                    (((mn_chunk & 7) ^ (k & 7)) << 4));
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
      :
      : "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// ---- mbarrier extras ------------------------------------------------------------
__device__ __forceinline__ void mbar_arrive(uint64_t* mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(mbar)) : "memory");
}

// ---- TMA ------------------------------------------------------------------------
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
// 2-D tile {x (inner), y} of tensor map `m` → shared `dst`, tx bytes on `mbar`
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* m, int x, int y,
                                            uint64_t* mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(smem_u32(mbar))
      : "memory");
}

// 2-D tile multicast to the CTAs of `mask` in the cluster: the same shared
// offset `dst` and mbarrier offset in each destination CTA
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* m, int x, int y,
                                               uint64_t* mbar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(smem_u32(mbar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// tcgen05.commit arriving on the mbarrier at the same offset in every CTA of `mask`
__device__ __forceinline__ void commit_mc(uint64_t* mbar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(mbar)), "h"(mask)
      : "memory");
}

// ---- CTA-pair (cta_group::2) forms ------------------------------------------
// shared::cluster address of the same shared variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
// TMA loads of a CTA pair: data to this CTA's smem, completion to the barrier at
// cluster address `mbar_cl` (the leader CTA's)
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* m, int x, int y,
                                                 uint32_t mbar_cl) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(mbar_cl)
      : "memory");
}
__device__ __forceinline__ void tma_im2col_4d_pair(void* dst, const CUtensorMap* m, int c, int w,
                                                   int h, int n, uint16_t ow, uint16_t oh,
                                                   uint32_t mbar_cl) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6], {%7, %8};" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c), "r"(w), "r"(h), "r"(n), "r"(mbar_cl), "h"(ow),
      "h"(oh)
      : "memory");
}
__device__ __forceinline__ void mma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void commit_pair(uint64_t* mbar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(mbar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t mbar_cl) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(mbar_cl)
               : "memory");
}
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}

// 4-D tile {c (inner), x, y, n} of a tiled tensor map (OOB → zero fill)
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* m, int c, int x, int y,
                                            int n, uint64_t* mbar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c), "r"(x), "r"(y), "r"(n), "r"(smem_u32(mbar))
      : "memory");
}

// 3-D tile {x (inner), y, z} of tensor map `m` → shared `dst`
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* m, int x, int y, int z,
                                            uint64_t* mbar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(mbar))
      : "memory");
}

// 4-D im2col box of tensor map `m` (NHWC: {c, w, h, n} base coordinates of the box's
// first pixel, filter offsets {ow, oh} added per pixel) → shared `dst`
__device__ __forceinline__ void tma_im2col_4d(void* dst, const CUtensorMap* m, int c, int w,
                                              int h, int n, uint16_t ow, uint16_t oh,
                                              uint64_t* mbar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6], {%7, %8};" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c), "r"(w), "r"(h), "r"(n), "r"(smem_u32(mbar)),
      "h"(ow), "h"(oh)
      : "memory");
}

// ---- cp.async (16 B, zero fill when !ok) ------------------------------------------
__device__ __forceinline__ void cp16(uint32_t dst, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(ok ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---- TMEM loads: 32 lanes x 16 columns (32x32b.x16) ---------------------------------
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 consecutive accumulator columns of this thread's lane, one wait
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&a)[16], float (&b)[16]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    a[i] = __uint_as_float(r[i]);
    b[i] = __uint_as_float(r[16 + i]);
  }
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Programmatic dependent launch gate (see cnn::pdl_gate): called by the conv
// GEMMs after their TMEM allocation, so a parked dependent CTA can never hold
// TMEM columns a running CTA of the chain still has to allocate.
__device__ __forceinline__ void pdl_gate() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

}  // namespace tc
