// Microbenchmark: cost of one pipelined-chunk iteration (cp.async wait +
// __syncthreads + refill + FFMA block) at 8 warps / SM, 1 CTA per SM, with
// and without thread-block clusters.  Build + run on the GPU box:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/lb tools/loop_bench.cu && /tmp/lb
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void cp16(void* s, const void* g) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(a), "l"(g));
}

template <int V>
__global__ void __launch_bounds__(256, 1) k(const float* __restrict__ src, float* out,
                                            long long* cyc, int iters) {
  extern __shared__ __align__(16) float sm[];
  const int tid = threadIdx.x;
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0.f;
  for (int e = tid; e < 4 * 4096; e += 256) sm[e] = 1e-3f * e;
  __syncthreads();
  long long t0 = clock64();
  for (int c = 0; c < iters; ++c) {
    if (V >= 1) asm volatile("cp.async.wait_group 2;\n" ::: "memory");
    __syncthreads();
    if (V == 6 || V == 7) {  // gathered rows (X-like) + strided 64 B segments (W-like)
      float* st = sm + (c & 3) * 4096;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int e = tid + 256 * j, r = e >> 4, q = e & 15;
        const size_t row = (size_t)((r * 7919 + blockIdx.x * 31) % 10000);
        cp16(st + r * 68 + 4 * q, src + row * 784 + c * 64 + 4 * q);
      }
      {
        const int k = tid >> 2, q = tid & 3;
        const float* w = V == 6 ? src + 8000000 + (size_t)(c * 64 + k) * 256 + blockIdx.x * 16 + 4 * q
                                : src + 8000000 + (size_t)(c * 64 + k) * 16 + 4 * q;
        cp16(st + 2176 + k * 20 + 4 * q, w);
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    if (V >= 2 && V <= 5) {
      float* st = sm + (c & 3) * 4096;
#pragma unroll
      for (int j = 0; j < 3; ++j)
        cp16(st + 4 * (tid + 256 * j), src + ((size_t)blockIdx.x * 64 + c) * 4096 + 4 * (tid + 256 * j));
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    if (V == 4 || V == 5) {
      const float* X = sm + ((c + 1) & 3) * 4096;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        float4 x[4], w[4];
        if (V == 4) {
#pragma unroll
          for (int i = 0; i < 4; ++i) x[i] = *reinterpret_cast<const float4*>(X + (tid & 7) * 68 + i * 8 * 68 + 8 * q);
#pragma unroll
          for (int i = 0; i < 4; ++i) w[i] = *reinterpret_cast<const float4*>(X + 2176 + (4 * q + i) * 20 + 4 * ((tid >> 3) & 3));
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i) { x[i] = make_float4(c * 1e-3f + i, q, i, 1.f); w[i] = make_float4(i, c * 1e-4f, q, 2.f); }
        }
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float xs[4] = {x[i].x, x[i].y, x[i].z, x[i].w};
            const float ws[4] = {w[kk].x, w[kk].y, w[kk].z, w[kk].w};
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[4 * i + j] = fmaf(xs[kk], ws[j], acc[4 * i + j]);
          }
      }
    }
    if (V == 3) {
      const float* X = sm + ((c + 1) & 3) * 4096;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        float4 x[4], w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) x[i] = *reinterpret_cast<const float4*>(X + (tid & 7) * 68 + i * 8 * 68 + 8 * q);
#pragma unroll
        for (int i = 0; i < 4; ++i) w[i] = *reinterpret_cast<const float4*>(X + 2176 + (4 * q + i) * 20 + 4 * ((tid >> 3) & 3));
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float xs[4] = {x[i].x, x[i].y, x[i].z, x[i].w};
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const float ws[4] = {w[kk].x, w[kk].y, w[kk].z, w[kk].w};
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[4 * i + j] = fmaf(xs[kk], ws[j], acc[4 * i + j]);
          }
        }
      }
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 12345.f) out[tid] = s;
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int V>
static void run(const char* name, int cluster, const float* src, float* out, long long* cyc) {
  const int smem = 200 * 1024, iters = 12;
  cudaFuncSetAttribute(k<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<V>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(32);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  for (int rep = 0; rep < 3; ++rep) cudaLaunchKernelEx(&cfg, k<V>, src, out, cyc, iters);
  cudaDeviceSynchronize();
  long long h[32];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double m = 0;
  for (int i = 0; i < 32; ++i) m += h[i];
  printf("%-34s cluster %2d: %7.1f cycles/iter  (%s)\n", name, cluster, m / 32 / iters,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  float *src, *out;
  long long* cyc;
  cudaMalloc(&src, (size_t)64 * 1024 * 1024 * 4);
  cudaMemset(src, 0, (size_t)64 * 1024 * 1024 * 4);
  cudaMalloc(&out, 4096);
  cudaMalloc(&cyc, 32 * 8);
  for (int cl : {1}) {
    run<0>("bar.sync", cl, src, out, cyc);
    run<1>("wait_group + bar.sync", cl, src, out, cyc);
    run<2>("+ 3 cp.async 16B refill", cl, src, out, cyc);
    run<3>("+ 2 quads (16 LDS.128, 128 FFMA)", cl, src, out, cyc);
    run<4>("+ 2 quads, k-outer FFMA order", cl, src, out, cyc);
    run<5>("+ 2 quads, register operands", cl, src, out, cyc);
    run<6>("gathered X rows + strided W (1KB)", cl, src, out, cyc);
    run<7>("gathered X rows + contiguous W", cl, src, out, cyc);
  }
  return 0;
}
