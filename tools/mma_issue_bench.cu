// tcgen05.mma issue cost: n back-to-back MMAs (M=128, N, K=8 tf32 or K=16 bf16) into 1..4
// accumulators, timed with clock64 (tools/ on one B200; DESIGN.md §3 quotes it):
//   nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2002_02885_b200/csrc \
//        tools/mma_issue_bench.cu -o tools/mmab.bin && tools/mmab.bin
#include <cstdio>
#include "pk_umma.cuh"
__global__ void k(unsigned long long* out, int N, int n, int bf16, int nacc) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tb;
  float* A = (float*)sm;            // 128 x 8 tf32 (4 KB) or 128 x 16 bf16 (4 KB)
  float* B = A + 128 * 8;           // N x 8
  for (int i = threadIdx.x; i < (128 + 256) * 8; i += blockDim.x) A[i] = 0.001f * (i % 7);
  if (threadIdx.x < 32) umma::tmem_alloc(&tb, 512);
  if (threadIdx.x == 0) { umma::mbar_init(&mbar, 1); umma::mbar_fence_init(); }
  umma::fence_async_smem();
  umma::fence_before(); __syncthreads(); umma::fence_after();
  if (threadIdx.x == 0) {
    uint32_t idesc = bf16 ? ((1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24))
                          : umma::idesc_tf32(128, N, false, false);
    uint64_t da = umma::kmaj_desc(umma::smem_u32(A), 128, 0), db = umma::kmaj_desc(umma::smem_u32(B), N, 0);
    long long c0 = clock64();
    for (int i = 0; i < n; ++i) {
      if (bf16) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
                     :: "r"(tb + (uint32_t)((i % nacc) * N)), "l"(da), "l"(db), "r"(idesc), "r"((uint32_t)(i >= nacc)));
      } else {
        umma::mma_tf32(tb + (uint32_t)((i % nacc) * N), da, db, idesc, i >= nacc);
      }
    }
    long long c1 = clock64();
    umma::commit(&mbar);
    umma::mbar_wait(&mbar, 0);
    long long c2 = clock64();
    out[0] = c1 - c0; out[1] = c2 - c0;
  }
  umma::fence_before(); __syncthreads();
  if (threadIdx.x < 32) umma::tmem_dealloc(tb, 512);
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 16);
  unsigned long long h[2];
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int bf = 0; bf < 2; ++bf)
    for (int N : {32, 64, 128})
      for (int nacc : {1, 2, 4}) {
        if (N * nacc > 512) continue;
        for (int rep = 0; rep < 2; ++rep) {
          k<<<1, 128, 64 * 1024>>>(d, N, 240, bf, nacc);
          cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        }
        printf("%s N=%3d acc=%d: issue %.1f cyc/mma, complete %.1f cyc/mma\n", bf ? "bf16 K=16" : "tf32 K=8 ", N, nacc, h[0] / 240.0, h[1] / 240.0);
      }
  cudaError_t e = cudaDeviceSynchronize(); printf("%s\n", cudaGetErrorString(e));
}
