// Microtest: does a tcgen05 K-major SW128 A descriptor whose start address is
// shifted by j rows (j*128 B, not 1024-aligned) read rows j..j+127 of a TMA-SW128
// tile — with base_offset 0, or with base_offset = j & 7?  (halo-tile conv idea)
//   nvcc -gencode arch=compute_100a,code=sm_100a -I../paper_2002_02885_b200/csrc \
//        -I../include tools/shift_test.cu -o /tmp/shift_test -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <vector>

#include "pk_tc.cuh"

__global__ void k(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
                  int shift, int boff, float* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar, done;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    umma::mbar_init(&bar, 1);
    umma::mbar_init(&done, 1);
    umma::mbar_fence_init();
  }
  if (warp == 0) umma::tmem_alloc(&slot, 64);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    umma::mbar_arrive_expect_tx(&bar, 256 * 128 + 64 * 128);
    tc::tma_load_2d(sm, &ma, 0, 0, &bar);
    tc::tma_load_2d(sm + 32768, &mb, 0, 0, &bar);
    umma::mbar_wait(&bar, 0);
    umma::fence_after();
    const uint32_t a = tc::smem_u32(sm) + shift * 128, b = tc::smem_u32(sm) + 32768;
    const uint32_t idesc = tc::idesc_bf16(128, 64, false, false);
    for (int ks = 0; ks < 4; ++ks) {
      uint64_t ad = tc::sdesc_sw128(a + ks * 32, 16, 1024);
      ad |= (uint64_t)(boff & 7) << 49;  // matrix base offset
      tc::mma_bf16(tmem, ad, tc::sdesc_sw128(b + ks * 32, 16, 1024), idesc, ks ? 1u : 0u);
    }
    umma::commit(&done);
  }
  __syncwarp();
  umma::mbar_wait(&done, 0);
  umma::fence_after();
  if (warp < 4) {
    const int row = warp * 32 + lane;
    for (int c = 0; c < 64; c += 16) {
      float v[16];
      tc::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
      for (int e = 0; e < 16; ++e) out[row * 64 + c + e] = v[e];
    }
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tmem, 64);
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  std::vector<__nv_bfloat16> A(256 * 64), B(64 * 64);
  std::vector<float> Af(256 * 64), Bf(64 * 64);
  for (int i = 0; i < 256 * 64; ++i) { float x = (float)((i * 7919) % 13 - 6) / 4.f; A[i] = __float2bfloat16(x); Af[i] = __bfloat162float(A[i]); }
  for (int i = 0; i < 64 * 64; ++i) { float x = (float)((i * 104729) % 11 - 5) / 4.f; B[i] = __float2bfloat16(x); Bf[i] = __bfloat162float(B[i]); }
  __nv_bfloat16 *dA, *dB; float* dO;
  cudaMalloc(&dA, A.size() * 2); cudaMalloc(&dB, B.size() * 2); cudaMalloc(&dO, 128 * 64 * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  CUtensorMap ma, mb;
  cuuint64_t da[2] = {64, 256}, sa[1] = {128}, db[2] = {64, 64}, sb[1] = {128};
  cuuint32_t ba[2] = {64, 256}, bb[2] = {64, 64}, es[2] = {1, 1};
  enc(&ma, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dA, da, sa, ba, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&mb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dB, db, sb, bb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  std::vector<float> O(128 * 64);
  for (int shift : {0, 1, 3, 8, 13, 58, 117}) {
    for (int mode = 0; mode < 2; ++mode) {
      const int boff = mode ? (shift & 7) : 0;
      k<<<1, 128, 48 * 1024>>>(ma, mb, shift, boff, dO);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
      double err = 0;
      for (int i = 0; i < 128; ++i)
        for (int n = 0; n < 64; ++n) {
          double r = 0;
          for (int kk = 0; kk < 64; ++kk) r += (double)Af[(i + shift) * 64 + kk] * Bf[n * 64 + kk];
          err = fmax(err, fabs(r - O[i * 64 + n]));
        }
      printf("shift %3d base_offset %d: max |err| %g %s\n", shift, boff, err, err < 1e-3 ? "OK" : "WRONG");
    }
  }
  return 0;
}
