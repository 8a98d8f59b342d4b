// Standalone check of the tcgen05 layer (pk_umma.cuh) on one B200:
//   C[128 x N] = A[128 x K] · B[K x N]   (A row-major (m,k), B row-major (k,n))
// staged into shared memory as K-major or MN-major canonical layouts, 1xTF32
// or 3xTF32, accumulated in TMEM, read back with tcgen05.ld.  Compares with
// a float64 host GEMM.  Build + run:
//   nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2002_02885_b200/csrc \
//        tools/umma_selftest.cu -o /tmp/umma_selftest && /tmp/umma_selftest
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "pk_umma.cuh"

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e = (x);                                                          \
    if (e != cudaSuccess) {                                                       \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);   \
      exit(1);                                                                    \
    }                                                                             \
  } while (0)

constexpr int M = 128;
constexpr int KC = 32;  // k per staged chunk (4 MMA K-steps)

template <bool A_MN, bool B_MN, bool X3>  // A_MN/B_MN unused (K-major only)
__global__ void k_gemm(const float* A, const float* B, float* C, int N, int K) {
  extern __shared__ __align__(128) unsigned char sm[];
  float* sAh = reinterpret_cast<float*>(sm);
  float* sAl = sAh + M * KC;
  float* sBh = sAl + M * KC;
  float* sBl = sBh + 256 * KC;
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  const uint32_t ncols = umma::tmem_cols_pow2(N);
  if (warp == 0) umma::tmem_alloc(&tbase, ncols);
  if (tid == 0) {
    umma::mbar_init(&mbar, 1);
    umma::mbar_fence_init();
  }
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = tbase;
  const uint32_t idesc = umma::idesc_tf32(M, N, A_MN, B_MN);
  uint32_t phase = 0;
  for (int k0 = 0; k0 < K; k0 += KC) {
    // stage A (M x KC) and B (N x KC as the MMA's B operand: rows = n)
    for (int e = tid; e < M * KC; e += blockDim.x) {
      const int m = e / KC, k = e % KC;
      const float v = A[(size_t)m * K + k0 + k];
      float h, l;
      if (X3) umma::split3(v, h, l); else { h = v; l = 0.f; }
      const uint32_t off = umma::kmaj_off(m, k, M);
      sAh[off / 4] = h;
      sAl[off / 4] = l;
    }
    for (int e = tid; e < N * KC; e += blockDim.x) {
      const int k = e / N, n = e % N;
      const float v = B[(size_t)(k0 + k) * N + n];
      float h, l;
      if (X3) umma::split3(v, h, l); else { h = v; l = 0.f; }
      const uint32_t off = umma::kmaj_off(n, k, N);
      sBh[off / 4] = h;
      sBl[off / 4] = l;
    }
    umma::fence_async_smem();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    if (tid == 0) {
      const uint32_t ah = umma::smem_u32(sAh), al = umma::smem_u32(sAl);
      const uint32_t bh = umma::smem_u32(sBh), bl = umma::smem_u32(sBl);
      for (int s = 0; s < KC / 8; ++s) {
        auto da = [&](uint32_t b) { return umma::kmaj_desc(b, M, s); };
        auto db = [&](uint32_t b) { return umma::kmaj_desc(b, N, s); };
        const bool acc = (k0 > 0) || (s > 0);
        umma::mma_tf32(tmem, da(ah), db(bh), idesc, acc);
        if (X3) {
          umma::mma_tf32(tmem, da(ah), db(bl), idesc, true);
          umma::mma_tf32(tmem, da(al), db(bh), idesc, true);
        }
      }
      umma::commit(&mbar);
    }
    umma::mbar_wait(&mbar, phase);
    phase ^= 1;
    umma::fence_after();
  }
  // epilogue: warp w ↔ TMEM lanes 32w..32w+31 = rows of C
  const int row = warp * 32 + (tid % 32);
  for (int c = 0; c < N; c += 8) {
    float v[8];
    umma::tmem_ld8(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
    umma::tmem_wait_ld();
    for (int i = 0; i < 8; ++i) C[(size_t)row * N + c + i] = v[i];
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tmem, ncols);
}

template <bool A_MN, bool B_MN, bool X3>  // A_MN/B_MN unused (K-major only)
static bool run(int N, int K, double tol) {
  std::vector<float> A((size_t)M * K), B((size_t)K * N), C((size_t)M * N);
  srand(1234 + N + K);
  for (auto& x : A) x = (rand() / (float)RAND_MAX - 0.5f) * 2.f;
  for (auto& x : B) x = (rand() / (float)RAND_MAX - 0.5f) * 2.f;
  float *dA, *dB, *dC;
  CK(cudaMalloc(&dA, A.size() * 4));
  CK(cudaMalloc(&dB, B.size() * 4));
  CK(cudaMalloc(&dC, C.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(dC, 0, C.size() * 4));
  const int smem = (2 * M * KC + 2 * 256 * KC) * 4;
  CK(cudaFuncSetAttribute(k_gemm<A_MN, B_MN, X3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_gemm<A_MN, B_MN, X3><<<1, 128, smem>>>(dA, dB, dC, N, K);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost));
  double maxrel = 0, maxabs = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0, mag = 0;
      for (int k = 0; k < K; ++k) {
        ref += (double)A[(size_t)m * K + k] * B[(size_t)k * N + n];
        mag += fabs((double)A[(size_t)m * K + k] * B[(size_t)k * N + n]);
      }
      const double d = fabs(C[(size_t)m * N + n] - ref);
      maxabs = fmax(maxabs, d);
      maxrel = fmax(maxrel, d / mag);
    }
  const bool ok = maxrel <= tol;
  printf("%-4s A_%s B_%s %s N=%3d K=%4d  max|err|=%.3e  max err/Σ|ab|=%.3e  %s\n", ok ? "OK" : "FAIL",
         A_MN ? "MN" : "K ", B_MN ? "MN" : "K ", X3 ? "3xTF32" : "1xTF32", N, K, maxabs, maxrel,
         ok ? "" : "<<<");
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dC);
  return ok;
}

int main() {
  bool ok = true;
  ok &= run<false, false, false>(32, 64, 2e-3);
  ok &= run<false, false, true>(32, 64, 1e-6);
  ok &= run<false, false, true>(64, 128, 1e-6);
  ok &= run<false, false, true>(128, 256, 1e-6);
  ok &= run<false, false, true>(256, 800, 1e-6);
  ok &= run<false, false, true>(16, 32, 1e-6);
  printf(ok ? "ALL OK\n" : "SOME FAILED\n");
  return ok ? 0 : 1;
}
