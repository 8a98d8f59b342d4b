// pk_cnn_ops.cuh — HBM-bound kernels of the conv pack path.
//
// Every kernel is grouped: one launch covers one layer of all members of the
// pack.  Problem descriptors (packtrain_b200.h pk_cnn_*) live in device memory;
// blk0[i] is the first block of problem i (prefix over problems, blk0[nprob] =
// grid size), so a block finds its problem by binary search and never mixes
// two members.  Tensors are NHWC bf16 with C a multiple of 8: a thread moves
// one 16-byte vector of 8 channels of one pixel row ("item").
//
// Determinism / K-invariance: every reduction (BN statistics, BN backward,
// bias and depthwise weight gradients, the softmax head) sums a fixed row
// partition of the member's own rows in a fixed order: per-block fp32 partial
// sums over `rpb` rows (chosen by the planner from the member's own row count)
// → workspace → a two-level ticket tree (tree_reduce) adds them in fp64 in
// block order.  Results depend only on the member's shape,
// never on which members share the launch, so packed == standalone bit for bit.
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

#include "packtrain_b200.h"

namespace cnn {

constexpr int kBlock = 256;

__device__ __forceinline__ int find_prob(const int* blk0, int nprob, int b) {
  int lo = 0, hi = nprob - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(blk0 + mid) <= b) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Up to kPack problems of one launch travel in the kernel parameters (constant
// bank): a block's problem lookup and descriptor reads are then cached
// constant loads instead of a dependent chain of global loads.
constexpr int kPack = 64;
template <class T>
struct Pack {
  int nprob;
  int blk0[kPack + 1];
  T p[kPack];
};
template <class T>
__device__ __forceinline__ int pack_prob(const Pack<T>& G, int b) {
  int lo = 0, hi = G.nprob - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (G.blk0[mid] <= b) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ void ld8(const void* p, float (&v)[8]) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ void st8(void* p, const float (&v)[8]) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = u;
}
__device__ __forceinline__ void ld8f(const float* p, float (&v)[8]) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p));
  const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ const uint8_t* bptr(const void* base, long long row, int ld, int ch) {
  return static_cast<const uint8_t*>(base) + (row * ld + ch) * 2;
}
__device__ __forceinline__ uint8_t* bptr(void* base, long long row, int ld, int ch) {
  return static_cast<uint8_t*>(base) + (row * ld + ch) * 2;
}

__device__ __forceinline__ float act_fwd(float x, int act) {
  if (act == PK_CNN_ACT_RELU) return fmaxf(x, 0.f);
  if (act == PK_CNN_ACT_RELU6) return fminf(fmaxf(x, 0.f), 6.f);
  return x;
}
// derivative of the activation, from its OUTPUT (relu: out > 0 ⇔ in > 0;
// relu6: 0 < out < 6 ⇔ 0 < in < 6 — torch's hardtanh_backward rule)
__device__ __forceinline__ float act_bwd(float out, int act) {
  if (act == PK_CNN_ACT_RELU) return out > 0.f ? 1.f : 0.f;
  if (act == PK_CNN_ACT_RELU6) return (out > 0.f && out < 6.f) ? 1.f : 0.f;
  return 1.f;
}

// ------------------------------------------------------------------------------
// Column (channel) partial sums of up to two per-element quantities over rows
// [r0, r1) of one block.  F(row, ch0, a[8], b[8]) fills the two values of the 8
// channels ch0.. of `row`.  Writes ws[blk][2][c].
// ------------------------------------------------------------------------------
template <class F>
__device__ __forceinline__ void col_partials(int r0, int r1, int c, int blk, float* ws, F f) {
  __shared__ float sh[2][2048];
  const int cgs = c >> 3;
  int cgp = 1;  // channel groups rounded up to a power of two (<= 256)
  while (cgp < cgs) cgp <<= 1;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int j = t & (cgp - 1), rl = t / cgp, nr = kBlock / cgp;
  float s1[8], s2[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) s1[e] = s2[e] = 0.f;
  if (j < cgs) {
#pragma unroll 4
    for (int r = r0 + rl; r < r1; r += nr) {
      float a[8], b[8];
      f(r, 8 * j, a, b);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        s1[e] += a[e];
        s2[e] += b[e];
      }
    }
  }
  if (cgp <= 32) {
    // lanes l, l ^ cgp, l ^ 2cgp, ... of a warp share channel group j: fixed xor tree
    for (int o = 16; o >= cgp; o >>= 1) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        s1[e] += __shfl_xor_sync(0xffffffffu, s1[e], o);
        s2[e] += __shfl_xor_sync(0xffffffffu, s2[e], o);
      }
    }
    if (lane < cgp && j < cgs) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        sh[0][warp * c + 8 * j + e] = s1[e];
        sh[1][warp * c + 8 * j + e] = s2[e];
      }
    }
    __syncthreads();
    float* out = ws + (long long)blk * 2 * c;
    for (int ch = t; ch < c; ch += kBlock) {
      float a = 0.f, b = 0.f;
#pragma unroll
      for (int w = 0; w < kBlock / 32; ++w) {
        a += sh[0][w * c + ch];
        b += sh[1][w * c + ch];
      }
      out[ch] = a;
      out[c + ch] = b;
    }
  } else {
    // nr (<= 4) row lanes, each a set of whole warps: combine through shared memory
    if (j < cgs) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        sh[0][rl * c + 8 * j + e] = s1[e];
        sh[1][rl * c + 8 * j + e] = s2[e];
      }
    }
    __syncthreads();
    float* out = ws + (long long)blk * 2 * c;
    for (int ch = t; ch < c; ch += kBlock) {
      float a = 0.f, b = 0.f;
      for (int l = 0; l < nr; ++l) {
        a += sh[0][l * c + ch];
        b += sh[1][l * c + ch];
      }
      out[ch] = a;
      out[c + ch] = b;
    }
  }
}

// Two-level fixed-order reduction of per-block partial records.
// Every block has written ws[blk*stride + i], i < nout.  Blocks form groups of
// kRedGroup; the last block of a group to arrive (atomic ticket on
// counters[1 + group]) sums its group's records in block order into an fp64
// group record; the last group reducer (ticket on counters[0]) sums the group
// records in group order into tot[0..nout) and returns true — in exactly one
// block.  Tickets reset themselves, so the counters are reusable (graph replay).
// Workspace layout: [nblk*stride floats][ngroups*nout doubles][nout doubles].
constexpr int kRedGroup = 16;
constexpr int kRedMaxBlocks = kRedGroup * kRedGroup;  // planner keeps nblk <= this

__device__ __forceinline__ bool ticket(int* counter, int n) {
  __shared__ int s_last;
  // the CTA barrier orders every thread's stores before thread 0's gpu-scope
  // fence + atomic (PTX release cumulativity), so one fence per block suffices
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const int prev = atomicAdd(counter, 1);
    s_last = (prev == n - 1);
    if (s_last) *counter = 0;
  }
  __syncthreads();
  if (s_last) __threadfence();
  return s_last != 0;
}

__device__ __forceinline__ bool tree_reduce(float* ws, int blk, int nblk, int nout, int stride,
                                            int* counters, double** tot_out) {
  const int ngroups = (nblk + kRedGroup - 1) / kRedGroup;
  const int grp = blk / kRedGroup;
  const int b0 = grp * kRedGroup, b1 = min(nblk, b0 + kRedGroup);
  double* grec = reinterpret_cast<double*>(ws + (((long long)nblk * stride + 1) & ~1LL));
  double* tot = grec + (long long)ngroups * nout;
  *tot_out = tot;
  if (!ticket(counters + 1 + grp, b1 - b0)) return false;
  for (int i = threadIdx.x; i < nout; i += kBlock) {
    double v = 0.0;
    for (int b = b0; b < b1; ++b) v += __ldcg(ws + (long long)b * stride + i);
    grec[(long long)grp * nout + i] = v;
  }
  if (!ticket(counters, ngroups)) return false;
  for (int i = threadIdx.x; i < nout; i += kBlock) {
    double v = 0.0;
    for (int g = 0; g < ngroups; ++g) v += __ldcg(grec + (long long)g * nout + i);
    tot[i] = v;
  }
  __syncthreads();
  return true;
}

// ============================== batch norm =====================================
__global__ void __launch_bounds__(kBlock, 3) k_bn_stats(const __grid_constant__ Pack<pk_cnn_bn> G) {
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_bn& P = G.p[pi];
  const int blk = blockIdx.x - G.blk0[pi], nblk = G.blk0[pi + 1] - G.blk0[pi];
  const int r0 = blk * P.rpb, r1 = min(P.rows, r0 + P.rpb);
  col_partials(r0, r1, P.c, blk, P.ws, [&](int r, int ch, float (&a)[8], float (&b)[8]) {
    ld8(bptr(P.x, r, P.ldx, ch), a);
#pragma unroll
    for (int e = 0; e < 8; ++e) b[e] = a[e] * a[e];
  });
  double* tot;
  if (!tree_reduce(P.ws, blk, nblk, 2 * P.c, 2 * P.c, P.counter, &tot)) return;
  for (int ch = threadIdx.x; ch < P.c; ch += kBlock) {
    const double mean = tot[ch] / P.rows;
    const double var = fmax(tot[P.c + ch] / P.rows - mean * mean, 0.0);
    P.stats[ch] = (float)mean;
    P.stats[P.c + ch] = (float)(1.0 / sqrt(var + (double)P.eps));
    if (P.run_mean) {
      const double unb = P.rows > 1 ? var * P.rows / (P.rows - 1) : var;
      P.run_mean[ch] = (float)((1.0 - P.momentum) * P.run_mean[ch] + P.momentum * mean);
      P.run_var[ch] = (float)((1.0 - P.momentum) * P.run_var[ch] + P.momentum * unb);
    }
  }
}

__device__ __forceinline__ void bn_coef(const pk_cnn_bn& P, int ch, float (&mean)[8],
                                        float (&rs)[8]) {
  if (P.use_running) {
    float v[8];
    ld8f(P.run_mean + ch, mean);
    ld8f(P.run_var + ch, v);
#pragma unroll
    for (int e = 0; e < 8; ++e) rs[e] = (float)(1.0 / sqrt((double)v[e] + (double)P.eps));
  } else {
    ld8f(P.stats + ch, mean);
    ld8f(P.stats + P.c + ch, rs);
  }
}

constexpr int kApplyRows = 2;  // rows per thread in the BN apply kernels

__global__ void __launch_bounds__(kBlock, 4) k_bn_apply(const __grid_constant__ Pack<pk_cnn_bn> G) {
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_bn& P = G.p[pi];
  const int cgs = P.c >> 3;
  const long long item = (long long)(blockIdx.x - G.blk0[pi]) * kBlock + threadIdx.x;
  const long long rg = item / cgs;  // group of kApplyRows rows
  if (rg * kApplyRows >= P.rows) return;
  const int ch = 8 * (int)(item - rg * cgs);
  float mean[8], rs[8], g[8], b[8];
  bn_coef(P, ch, mean, rs);
  ld8f(P.gamma + ch, g);
  ld8f(P.beta + ch, b);
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    g[e] *= rs[e];
    b[e] -= mean[e] * g[e];  // y = x·(γ·rstd) + (β − mean·γ·rstd)
  }
  const long long r0 = rg * kApplyRows;
  const int nr = (int)min((long long)kApplyRows, P.rows - r0);
  float x[kApplyRows][8], res[kApplyRows][8];
#pragma unroll
  for (int i = 0; i < kApplyRows; ++i)
    if (i < nr) {
      ld8(bptr(P.x, r0 + i, P.ldx, ch), x[i]);
      if (P.res) ld8(bptr(P.res, r0 + i, P.ldr, ch), res[i]);
    }
#pragma unroll
  for (int i = 0; i < kApplyRows; ++i)
    if (i < nr) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        float y = fmaf(x[i][e], g[e], b[e]);
        if (P.res) y += res[i][e];
        x[i][e] = act_fwd(y, P.act);
      }
      st8(bptr(P.out, r0 + i, P.ldo, ch), x[i]);
    }
}

// g = dout · act'(fout); xhat = (x - mean)·rstd
__device__ __forceinline__ void bn_g_xhat(const pk_cnn_bn& P, long long r, int ch, float (&g)[8],
                                          float (&xh)[8]) {
  float d[8], fo[8], x[8], mean[8], rs[8];
  ld8(bptr(P.dout, r, P.ldd, ch), d);
  ld8(bptr(P.x, r, P.ldx, ch), x);
  ld8f(P.stats + ch, mean);
  ld8f(P.stats + P.c + ch, rs);
  if (P.act != PK_CNN_ACT_NONE) ld8(bptr(P.fout, r, P.ldo, ch), fo);
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    g[e] = P.act != PK_CNN_ACT_NONE ? d[e] * act_bwd(fo[e], P.act) : d[e];
    xh[e] = (x[e] - mean[e]) * rs[e];
  }
}

__global__ void __launch_bounds__(kBlock, 3) k_bn_bwd_reduce(const __grid_constant__ Pack<pk_cnn_bn> G) {
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_bn& P = G.p[pi];
  const int blk = blockIdx.x - G.blk0[pi], nblk = G.blk0[pi + 1] - G.blk0[pi];
  const int r0 = blk * P.rpb, r1 = min(P.rows, r0 + P.rpb);
  col_partials(r0, r1, P.c, blk, P.ws, [&](int r, int ch, float (&a)[8], float (&b)[8]) {
    float xh[8];
    bn_g_xhat(P, r, ch, a, xh);
#pragma unroll
    for (int e = 0; e < 8; ++e) b[e] = a[e] * xh[e];
  });
  double* tot;
  if (!tree_reduce(P.ws, blk, nblk, 2 * P.c, 2 * P.c, P.counter, &tot)) return;
  bool bad = false;
  for (int ch = threadIdx.x; ch < P.c; ch += kBlock) {
    const double s1 = tot[ch], s2 = tot[P.c + ch];
    P.dbeta[ch] = (float)s1;
    P.dgamma[ch] = (float)s2;
    P.stats[2 * P.c + ch] = (float)(s1 / P.rows);
    P.stats[3 * P.c + ch] = (float)(s2 / P.rows);
    bad |= !isfinite(s1) || !isfinite(s2);
  }
  if (bad) *P.flag = 1;
}

__global__ void __launch_bounds__(kBlock, 2) k_bn_bwd_apply(const __grid_constant__ Pack<pk_cnn_bn> G) {
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_bn& P = G.p[pi];
  const int cgs = P.c >> 3;
  const long long item = (long long)(blockIdx.x - G.blk0[pi]) * kBlock + threadIdx.x;
  const long long rg = item / cgs;
  if (rg * kApplyRows >= P.rows) return;
  const int ch = 8 * (int)(item - rg * cgs);
  // dx = γ·rstd·(g − mean(g) − xhat·mean(g·xhat)) = ca·g + cb·x + cc per channel
  float ca[8], cb[8], cc[8];
  {
    float ga[8], mg[8], mgx[8], rs[8], mean[8];
    ld8f(P.gamma + ch, ga);
    ld8f(P.stats + ch, mean);
    ld8f(P.stats + P.c + ch, rs);
    ld8f(P.stats + 2 * P.c + ch, mg);
    ld8f(P.stats + 3 * P.c + ch, mgx);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      ca[e] = ga[e] * rs[e];
      cb[e] = -ca[e] * rs[e] * mgx[e];
      cc[e] = -ca[e] * mg[e] - cb[e] * mean[e];
    }
  }
  const long long r0 = rg * kApplyRows;
  const int nr = (int)min((long long)kApplyRows, P.rows - r0);
  const bool act = P.act != PK_CNN_ACT_NONE;
  // all loads of the thread's rows first (memory-level parallelism), then math
  float d[kApplyRows][8], x[kApplyRows][8], fo[kApplyRows][8];
#pragma unroll
  for (int i = 0; i < kApplyRows; ++i)
    if (i < nr) {
      ld8(bptr(P.dout, r0 + i, P.ldd, ch), d[i]);
      ld8(bptr(P.x, r0 + i, P.ldx, ch), x[i]);
      if (act) ld8(bptr(P.fout, r0 + i, P.ldo, ch), fo[i]);
    }
#pragma unroll
  for (int i = 0; i < kApplyRows; ++i) {
    if (i >= nr) break;
    const long long r = r0 + i;
    float dx[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float g = act ? d[i][e] * act_bwd(fo[i][e], P.act) : d[i][e];
      dx[e] = fmaf(ca[e], g, fmaf(cb[e], x[i][e], cc[e]));
      d[i][e] = g;
    }
    if (P.accumulate) {
      float o[8];
      ld8(bptr(P.dx, r, P.ldx2, ch), o);
#pragma unroll
      for (int e = 0; e < 8; ++e) dx[e] += o[e];
    }
    st8(bptr(P.dx, r, P.ldx2, ch), dx);
    if (P.dres) {
      if (P.res_accumulate) {
        float o[8];
        ld8(bptr(P.dres, r, P.ldr, ch), o);
#pragma unroll
        for (int e = 0; e < 8; ++e) d[i][e] += o[e];
      }
      st8(bptr(P.dres, r, P.ldr, ch), d[i]);
    }
  }
}

// ============================ depthwise conv =====================================
__global__ void __launch_bounds__(kBlock) k_dw_fprop(const __grid_constant__ Pack<pk_cnn_dw> G) {
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_dw& P = G.p[pi];
  const int cgs = P.c >> 3;
  const long long item = (long long)(blockIdx.x - G.blk0[pi]) * kBlock + threadIdx.x;
  const long long M = (long long)P.n * P.p * P.q;
  if (item >= M * cgs) return;
  const long long m = item / cgs;
  const int ch = 8 * (int)(item - m * cgs);
  const int n = (int)(m / (P.p * P.q)), rem = (int)(m - (long long)n * P.p * P.q);
  const int oy = rem / P.q, ox = rem - oy * P.q;
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  for (int r = 0; r < P.r; ++r) {
    const int iy = oy * P.stride - P.pad + r;
    if ((unsigned)iy >= (unsigned)P.h) continue;
    for (int s = 0; s < P.s; ++s) {
      const int ix = ox * P.stride - P.pad + s;
      if ((unsigned)ix >= (unsigned)P.w) continue;
      float x[8], w[8];
      ld8(bptr(P.x, ((long long)n * P.h + iy) * P.w + ix, P.ldx, ch), x);
      ld8(bptr(P.wt, r * P.s + s, P.c, ch), w);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = fmaf(x[e], w[e], acc[e]);
    }
  }
  st8(bptr(P.y, m, P.ldy, ch), acc);
}

__global__ void __launch_bounds__(kBlock) k_dw_dgrad(const __grid_constant__ Pack<pk_cnn_dw> G) {
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_dw& P = G.p[pi];
  const int cgs = P.c >> 3;
  const long long item = (long long)(blockIdx.x - G.blk0[pi]) * kBlock + threadIdx.x;
  const long long M = (long long)P.n * P.h * P.w;
  if (item >= M * cgs) return;
  const long long m = item / cgs;
  const int ch = 8 * (int)(item - m * cgs);
  const int n = (int)(m / (P.h * P.w)), rem = (int)(m - (long long)n * P.h * P.w);
  const int iy = rem / P.w, ix = rem - iy * P.w;
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  for (int r = 0; r < P.r; ++r) {
    const int ty = iy + P.pad - r;
    if (ty < 0 || ty % P.stride) continue;
    const int oy = ty / P.stride;
    if (oy >= P.p) continue;
    for (int s = 0; s < P.s; ++s) {
      const int tx = ix + P.pad - s;
      if (tx < 0 || tx % P.stride) continue;
      const int ox = tx / P.stride;
      if (ox >= P.q) continue;
      float d[8], w[8];
      ld8(bptr(P.dy, ((long long)n * P.p + oy) * P.q + ox, P.ldy, ch), d);
      ld8(bptr(P.wt, r * P.s + s, P.c, ch), w);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = fmaf(d[e], w[e], acc[e]);
    }
  }
  st8(bptr(P.y, m, P.ldx, ch), acc);
}

// Σ over a block's row lanes of each thread's 8-channel vector v (thread t owns
// channel group t % cgp of row lane t / cgp, cgp = pow2 >= c/8), written to
// out[0..c): fixed xor-shuffle tree inside warps, then warps / lanes in order.
__device__ __forceinline__ void lane_sum8(float (&v)[8], int c, int cgs, int cgp, float* sh,
                                          float* out) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int j = t & (cgp - 1), rl = t / cgp, nr = kBlock / cgp;
  int parts;
  if (cgp <= 32) {
    for (int o = 16; o >= cgp; o >>= 1) {
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] += __shfl_xor_sync(0xffffffffu, v[e], o);
    }
    if (lane < cgp && j < cgs) {
#pragma unroll
      for (int e = 0; e < 8; ++e) sh[warp * c + 8 * j + e] = v[e];
    }
    parts = kBlock / 32;
  } else {
    if (j < cgs) {
#pragma unroll
      for (int e = 0; e < 8; ++e) sh[rl * c + 8 * j + e] = v[e];
    }
    parts = nr;
  }
  __syncthreads();
  for (int ch = t; ch < c; ch += kBlock) {
    float a = 0.f;
    for (int w = 0; w < parts; ++w) a += sh[w * c + ch];
    out[ch] = a;
  }
  __syncthreads();
}

// dw[tap][c] = Σ_pix dy[pix][c] · x[im2col(pix, tap)][c]
__global__ void __launch_bounds__(kBlock) k_dw_wgrad(const __grid_constant__ Pack<pk_cnn_dw> G) {
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_dw& P = G.p[pi];
  const int blk = blockIdx.x - G.blk0[pi], nblk = G.blk0[pi + 1] - G.blk0[pi];
  const int taps = P.r * P.s;  // <= 9
  const int cgs = P.c >> 3;
  int cgp = 1;
  while (cgp < cgs) cgp <<= 1;
  const int t = threadIdx.x, j = t & (cgp - 1), rl = t / cgp, nr = kBlock / cgp, ch = 8 * j;
  const int pq = P.p * P.q;
  const long long M = (long long)P.n * pq;
  const long long m0 = (long long)blk * P.ppb, m1 = min(M, m0 + P.ppb);
  float acc[9][8];
#pragma unroll
  for (int k = 0; k < 9; ++k)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[k][e] = 0.f;
  if (j < cgs) {
    for (long long m = m0 + rl; m < m1; m += nr) {
      const int n = (int)(m / pq), rem = (int)(m - (long long)n * pq);
      const int oy = rem / P.q, ox = rem - oy * P.q;
      float d[8];
      ld8(bptr(P.dy, m, P.ldy, ch), d);
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        if (k >= taps) break;
        const int r = k / P.s, s = k - r * P.s;
        const int iy = oy * P.stride - P.pad + r, ix = ox * P.stride - P.pad + s;
        if ((unsigned)iy >= (unsigned)P.h || (unsigned)ix >= (unsigned)P.w) continue;
        float x[8];
        ld8(bptr(P.x, ((long long)n * P.h + iy) * P.w + ix, P.ldx, ch), x);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[k][e] = fmaf(d[e], x[e], acc[k][e]);
      }
    }
  }
  __shared__ float sh[2048];
  float* out = P.ws + (long long)blk * taps * P.c;
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    if (k >= taps) break;
    lane_sum8(acc[k], P.c, cgs, cgp, sh, out + k * P.c);
  }
  const int nout = taps * P.c;
  double* tot;
  if (!tree_reduce(P.ws, blk, nblk, nout, nout, P.counter, &tot)) return;
  bool bad = false;
  for (int i = threadIdx.x; i < nout; i += kBlock) {
    P.dw[i] = (float)tot[i];
    bad |= !isfinite(tot[i]);
  }
  if (bad) *P.flag = 1;
}

// ================================ pooling ========================================
// Bodies are templates on the window / stride (0 = runtime value) so the
// common shapes (3x3/2 ResNet stem, 2x2/2 LeNet) unroll their tap loops.
template <int R_, int S_, int ST_>
__device__ __forceinline__ void maxpool_fwd_item(const pk_cnn_pool& P, long long m, int ch) {
  const int R = R_ ? R_ : P.r, S = S_ ? S_ : P.s, ST = ST_ ? ST_ : P.stride;
  const int n = (int)(m / (P.p * P.q)), rem = (int)(m - (long long)n * P.p * P.q);
  const int oy = rem / P.q, ox = rem - oy * P.q;
  float best[8];
  uint8_t arg[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    best[e] = -INFINITY;
    arg[e] = 0;
  }
#pragma unroll
  for (int r = 0; r < (R_ ? R_ : 1); ++r) {
    for (int rr = r; rr < R; rr += (R_ ? R : 1)) {
      const int iy = oy * ST - P.pad + rr;
      if ((unsigned)iy >= (unsigned)P.h) continue;
#pragma unroll
      for (int s = 0; s < (S_ ? S_ : 1); ++s) {
        for (int ss = s; ss < S; ss += (S_ ? S : 1)) {
          const int ix = ox * ST - P.pad + ss;
          if ((unsigned)ix >= (unsigned)P.w) continue;
          float x[8];
          ld8(bptr(P.x, ((long long)n * P.h + iy) * P.w + ix, P.ldx, ch), x);
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (x[e] > best[e]) {
              best[e] = x[e];
              arg[e] = (uint8_t)(rr * S + ss);
            }
        }
      }
    }
  }
  st8(bptr(P.y, m, P.ldy, ch), best);
  uint2 a;
  a.x = arg[0] | (arg[1] << 8) | (arg[2] << 16) | ((uint32_t)arg[3] << 24);
  a.y = arg[4] | (arg[5] << 8) | (arg[6] << 16) | ((uint32_t)arg[7] << 24);
  *reinterpret_cast<uint2*>(P.arg + m * P.c + ch) = a;
}

// input pixel (iy, ix) receives dy of every window whose argmax is its tap
template <int R_, int S_, int ST_, bool AVG>
__device__ __forceinline__ void pool_bwd_item(const pk_cnn_pool& P, long long m, int ch) {
  const int R = R_ ? R_ : P.r, S = S_ ? S_ : P.s, ST = ST_ ? ST_ : P.stride;
  const int n = (int)(m / (P.h * P.w)), rem = (int)(m - (long long)n * P.h * P.w);
  const int iy = rem / P.w, ix = rem - iy * P.w;
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
#pragma unroll
  for (int r = 0; r < (R_ ? R_ : 1); ++r) {
    for (int rr = r; rr < R; rr += (R_ ? R : 1)) {
      const int ty = iy + P.pad - rr;
      if (ty < 0 || ty % ST) continue;
      const int oy = ty / ST;
      if (oy >= P.p) continue;
#pragma unroll
      for (int s = 0; s < (S_ ? S_ : 1); ++s) {
        for (int ss = s; ss < S; ss += (S_ ? S : 1)) {
          const int tx = ix + P.pad - ss;
          if (tx < 0 || tx % ST) continue;
          const int ox = tx / ST;
          if (ox >= P.q) continue;
          const long long o = ((long long)n * P.p + oy) * P.q + ox;
          float d[8];
          ld8(bptr(P.dy, o, P.ldy, ch), d);
          if (AVG) {
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[e] += d[e];
          } else {
            const uint2 a = *reinterpret_cast<const uint2*>(P.arg + o * P.c + ch);
            const uint8_t* ab = reinterpret_cast<const uint8_t*>(&a);
            const int tap = rr * S + ss;
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (ab[e] == tap) acc[e] += d[e];
          }
        }
      }
    }
  }
  if (AVG) {
    const float inv = 1.f / (float)(R * S);
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] *= inv;
  }
  if (P.accumulate) {
    float o[8];
    ld8(bptr(P.dx, m, P.ldx, ch), o);
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] += o[e];
  }
  st8(bptr(P.dx, m, P.ldx, ch), acc);
}

__global__ void __launch_bounds__(kBlock) k_maxpool_fwd(const __grid_constant__ Pack<pk_cnn_pool> G) {
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_pool& P = G.p[pi];
  const int cgs = P.c >> 3;
  const long long item = (long long)(blockIdx.x - G.blk0[pi]) * kBlock + threadIdx.x;
  if (item >= (long long)P.n * P.p * P.q * cgs) return;
  const long long m = item / cgs;
  const int ch = 8 * (int)(item - m * cgs);
  if (P.r == 3 && P.s == 3 && P.stride == 2) maxpool_fwd_item<3, 3, 2>(P, m, ch);
  else if (P.r == 2 && P.s == 2 && P.stride == 2) maxpool_fwd_item<2, 2, 2>(P, m, ch);
  else maxpool_fwd_item<0, 0, 0>(P, m, ch);
}

__global__ void __launch_bounds__(kBlock) k_maxpool_bwd(const __grid_constant__ Pack<pk_cnn_pool> G) {
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_pool& P = G.p[pi];
  const int cgs = P.c >> 3;
  const long long item = (long long)(blockIdx.x - G.blk0[pi]) * kBlock + threadIdx.x;
  if (item >= (long long)P.n * P.h * P.w * cgs) return;
  const long long m = item / cgs;
  const int ch = 8 * (int)(item - m * cgs);
  if (P.r == 3 && P.s == 3 && P.stride == 2) pool_bwd_item<3, 3, 2, false>(P, m, ch);
  else if (P.r == 2 && P.s == 2 && P.stride == 2) pool_bwd_item<2, 2, 2, false>(P, m, ch);
  else pool_bwd_item<0, 0, 0, false>(P, m, ch);
}

// average pool; the global case (window = the whole map) splits each output's
// window over kPoolLanes threads and combines them with a fixed xor tree
constexpr int kPoolLanes = 8;
__global__ void __launch_bounds__(kBlock) k_avgpool_fwd(const __grid_constant__ Pack<pk_cnn_pool> G) {
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_pool& P = G.p[pi];
  const int cgs = P.c >> 3;
  const bool global = P.r == P.h && P.s == P.w && P.pad == 0 && P.p == 1 && P.q == 1;
  const int lanes = global ? kPoolLanes : 1;
  const long long item = ((long long)(blockIdx.x - G.blk0[pi]) * kBlock + threadIdx.x) / lanes;
  const int lane = threadIdx.x % lanes;
  const long long total = (long long)P.n * P.p * P.q * cgs;
  const long long m = item / cgs;
  const int ch = 8 * (int)(item - m * cgs);
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  if (global) {
    const int hw = P.h * P.w;
    if (item < total)
      for (int i = lane; i < hw; i += lanes) {
        float x[8];
        ld8(bptr(P.x, m * hw + i, P.ldx, ch), x);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += x[e];
      }
#pragma unroll
    for (int o = kPoolLanes / 2; o; o >>= 1)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
    if (item >= total || lane != 0) return;
  } else {
    if (item >= total) return;
    const int n = (int)(m / (P.p * P.q)), rem = (int)(m - (long long)n * P.p * P.q);
    const int oy = rem / P.q, ox = rem - oy * P.q;
    for (int r = 0; r < P.r; ++r) {
      const int iy = oy * P.stride - P.pad + r;
      if ((unsigned)iy >= (unsigned)P.h) continue;
      for (int s = 0; s < P.s; ++s) {
        const int ix = ox * P.stride - P.pad + s;
        if ((unsigned)ix >= (unsigned)P.w) continue;
        float x[8];
        ld8(bptr(P.x, ((long long)n * P.h + iy) * P.w + ix, P.ldx, ch), x);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += x[e];
      }
    }
  }
  const float inv = 1.f / (float)(P.r * P.s);
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] *= inv;
  st8(bptr(P.y, m, P.ldy, ch), acc);
}

__global__ void __launch_bounds__(kBlock) k_avgpool_bwd(const __grid_constant__ Pack<pk_cnn_pool> G) {
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_pool& P = G.p[pi];
  const int cgs = P.c >> 3;
  const long long item = (long long)(blockIdx.x - G.blk0[pi]) * kBlock + threadIdx.x;
  if (item >= (long long)P.n * P.h * P.w * cgs) return;
  const long long m = item / cgs;
  const int ch = 8 * (int)(item - m * cgs);
  if (P.r == 2 && P.s == 2 && P.stride == 2) pool_bwd_item<2, 2, 2, true>(P, m, ch);
  else pool_bwd_item<0, 0, 0, true>(P, m, ch);
}

// ======================== softmax cross-entropy head ============================
// one block per member; reference engine.py:211-230 (loss) and :252-264 (dlogits)
__global__ void __launch_bounds__(kBlock) k_xent(const __grid_constant__ Pack<pk_cnn_head> G) {
  const pk_cnn_head& P = G.p[blockIdx.x];
  extern __shared__ float xs[];
  float* rmax = xs;
  float* rsum = xs + P.rows;
  float* rloss = xs + 2 * P.rows;
  int* rlab = reinterpret_cast<int*>(xs + 3 * P.rows);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float inv = 1.f / (float)P.rows;
  for (int r = warp; r < P.rows; r += kBlock / 32) {
    const float* z = P.logits + (long long)r * P.ldl;
    float mx = -INFINITY;
    for (int j = lane; j < P.classes; j += 32) mx = fmaxf(mx, z[j]);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float se = 0.f;
    for (int j = lane; j < P.classes; j += 32) se += expf(z[j] - mx);
#pragma unroll
    for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
    const long long lab = P.labels[P.idx ? P.idx[r] : r];
    if (lane == 0) {
      rmax[r] = mx;
      rsum[r] = se;
      rlab[r] = (int)lab;
      rloss[r] = logf(se) - (z[lab] - mx);
    }
    if (P.dlogits) {
      const float is = 1.f / se;
      __nv_bfloat16* d = static_cast<__nv_bfloat16*>(P.dlogits) + (long long)r * P.ldl;
      for (int j = lane; j < P.ldl; j += 32) {
        float v = 0.f;
        if (j < P.classes) v = (expf(z[j] - mx) * is - (j == lab ? 1.f : 0.f)) * inv;
        d[j] = __float2bfloat16_rn(v);
      }
    }
  }
  __syncthreads();
  bool bad = false;
  if (P.dbias) {
    for (int j = threadIdx.x; j < P.classes; j += kBlock) {
      float s = 0.f;
      for (int r = 0; r < P.rows; ++r) {
        const float z = P.logits[(long long)r * P.ldl + j];
        s += (expf(z - rmax[r]) / rsum[r] - (j == rlab[r] ? 1.f : 0.f)) * inv;
      }
      P.dbias[j] = s;
      bad |= !isfinite(s);
    }
  }
  if (threadIdx.x == 0) {
    double l = 0.0;
    for (int r = 0; r < P.rows; ++r) l += rloss[r];
    l /= P.rows;
    *P.loss = (float)l;
    bad |= !isfinite(l);
  }
  if (bad && P.flag) *P.flag = 1;
}

// =================== bias + activation backward (LeNet layers) =====================
__global__ void __launch_bounds__(kBlock, 3) k_bias_act_bwd(const __grid_constant__ Pack<pk_cnn_bias> G) {
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_bias& P = G.p[pi];
  const int blk = blockIdx.x - G.blk0[pi], nblk = G.blk0[pi + 1] - G.blk0[pi];
  const int r0 = blk * P.rpb, r1 = min(P.rows, r0 + P.rpb);
  col_partials(r0, r1, P.c, blk, P.ws, [&](int r, int ch, float (&a)[8], float (&b)[8]) {
    ld8(bptr(P.dy, r, P.ld, ch), a);
    if (P.act != PK_CNN_ACT_NONE) {
      float fo[8];
      ld8(bptr(P.fout, r, P.ld, ch), fo);
#pragma unroll
      for (int e = 0; e < 8; ++e) a[e] *= act_bwd(fo[e], P.act);
    }
    if (P.act != PK_CNN_ACT_NONE || P.g != P.dy) st8(bptr(P.g, r, P.ld, ch), a);
#pragma unroll
    for (int e = 0; e < 8; ++e) b[e] = 0.f;
  });
  double* tot;
  if (!tree_reduce(P.ws, blk, nblk, P.c, 2 * P.c, P.counter, &tot)) return;
  bool bad = false;
  for (int ch = threadIdx.x; ch < P.c; ch += kBlock) {
    P.dbias[ch] = (float)tot[ch];
    bad |= !isfinite(tot[ch]);
  }
  if (bad) *P.flag = 1;
}

// ========================== WGRAD split reduction ================================
__global__ void __launch_bounds__(kBlock) k_split_reduce(const __grid_constant__ Pack<pk_cnn_reduce> G) {
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_reduce& P = G.p[pi];
  const long long i4 = (long long)(blockIdx.x - G.blk0[pi]) * kBlock + threadIdx.x;
  if (i4 * 4 >= P.len) return;
  float4 s = __ldcg(reinterpret_cast<const float4*>(P.src) + i4);
  for (int j = 1; j < P.splits; ++j) {
    const float4 v = __ldcg(reinterpret_cast<const float4*>(P.src + (long long)j * P.len) + i4);
    s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
  }
  reinterpret_cast<float4*>(P.dst)[i4] = s;
  if (!isfinite(s.x) || !isfinite(s.y) || !isfinite(s.z) || !isfinite(s.w)) *P.flag = 1;
}

// ====================== fused multi-member optimizer (K7) ==========================
// reference engine.py:295-326 (+ coupled weight decay g += wd·w, the torch.optim
// rule, as the north_star's per-member extension).  A flagged member (non-finite
// gradient anywhere) is left untouched, engine.py:297-299.
constexpr int kOptChunk = 4096;  // elements per block
__global__ void __launch_bounds__(kBlock) k_opt(const pk_cnn_opt_seg* segs, const int* blk0,
                                                int nseg) {
  const int si = find_prob(blk0, nseg, blockIdx.x);
  const pk_cnn_opt_seg& S = segs[si];
  if (*S.flag) return;  // the member's commit verdict (k_commit mode 0)
  const long long base = (long long)(blockIdx.x - blk0[si]) * kOptChunk;
  const int t = *S.step + 1;
  float c1 = 1.f, c2 = 1.f;
  if (S.kind == PK_OPT_ADAM) {
    c1 = (float)(1.0 - pow(0.9, (double)t));
    c2 = (float)(1.0 - pow(0.999, (double)t));
  }
  const float lr = S.lr, wd = S.wd;
  for (int k = threadIdx.x; k < kOptChunk; k += kBlock) {
    const long long i = base + k;
    if (i >= S.len) break;
    float w = S.w[i];
    float g = S.g[i];
    if (wd != 0.f) g = fmaf(wd, w, g);
    switch (S.kind) {
      case PK_OPT_SGD:
        w -= lr * g;
        break;
      case PK_OPT_MOMENTUM: {
        const float v = 0.9f * S.s1[i] + g;
        S.s1[i] = v;
        w -= lr * v;
        break;
      }
      case PK_OPT_ADAGRAD: {
        const float a = S.s1[i] + g * g;
        S.s1[i] = a;
        w -= lr * g / (sqrtf(a) + 1e-10f);
        break;
      }
      default: {  // adam
        const float m = 0.9f * S.s1[i] + 0.1f * g;
        const float v = 0.999f * S.s2[i] + 0.001f * (g * g);
        S.s1[i] = m;
        S.s2[i] = v;
        w -= lr * (m / c1) / (sqrtf(v / c2) + 1e-8f);
      }
    }
    S.w[i] = w;
    if (S.w16) static_cast<__nv_bfloat16*>(S.w16)[i] = __float2bfloat16_rn(w);
  }
}

// ================= transposed bf16 weights for DGRAD (B operand) ===================
__global__ void __launch_bounds__(kBlock) k_publish_t(const __grid_constant__ Pack<pk_cnn_tpose> G) {
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_tpose& P = G.p[pi];
  const int tk = (P.k + 31) / 32, tc = (P.c + 31) / 32;
  int b = blockIdx.x - G.blk0[pi];
  const int tap = b / (tk * tc);
  b -= tap * tk * tc;
  const int kt = b / tc, ct = b - kt * tc;
  __shared__ uint16_t tile[32][33];
  const uint16_t* src = static_cast<const uint16_t*>(P.src);
  uint16_t* dst = static_cast<uint16_t*>(P.dst);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int i = ty; i < 32; i += 8) {
    const int co = kt * 32 + i, ci = ct * 32 + tx;
    tile[i][tx] = (co < P.k && ci < P.c) ? src[(long long)co * P.kpad + tap * P.c + ci] : 0;
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int ci = ct * 32 + i, co = kt * 32 + tx;
    if (ci < P.c && co < P.k) dst[(long long)ci * P.kpadt + tap * P.k + co] = tile[tx][i];
  }
}

// Commit, reference packing.py:250-257 + engine.py:297-299: members are
// updated in pack order and the first non-finite gradient aborts the loop, so a
// member commits only if no member at or before it (in the problem order) is
// flagged.  mode 0 (before the optimizer, one thread): verdict = prefix-OR of
// the flags; mode 1 (after it): step += !verdict, verdict |= flag << 1, flag = 0.
__global__ void k_commit(const pk_cnn_commit* probs, int nprob, int mode) {
  if (mode == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      int run = 0;
      for (int i = 0; i < nprob; ++i) {
        run |= *probs[i].flag;
        *probs[i].verdict = run ? 1 : 0;
      }
    }
    return;
  }
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nprob) return;
  const pk_cnn_commit& P = probs[i];
  const int eff = *P.verdict;
  if (!eff) *P.step += 1;
  *P.verdict = eff | ((*P.flag ? 1 : 0) << 1);
  *P.flag = 0;
}

// batch gather: one block per 4 KB of rows, 16-byte vectors
constexpr int kGatherChunk = 4096;
__global__ void __launch_bounds__(kBlock) k_gather(const __grid_constant__ Pack<pk_cnn_gather> G) {
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_gather& P = G.p[pi];
  const long long v0 = (long long)(blockIdx.x - G.blk0[pi]) * (kGatherChunk / 16);
  const long long vrow = P.row_bytes / 16, total = vrow * P.rows;
  for (long long v = v0 + threadIdx.x; v < min(total, v0 + kGatherChunk / 16); v += kBlock) {
    const long long r = v / vrow, c = v - r * vrow;
    const uint4* s = reinterpret_cast<const uint4*>(static_cast<const uint8_t*>(P.src) +
                                                    P.idx[r] * P.row_bytes) + c;
    reinterpret_cast<uint4*>(static_cast<uint8_t*>(P.dst) + r * P.row_bytes)[c] = *s;
  }
}

}  // namespace cnn
