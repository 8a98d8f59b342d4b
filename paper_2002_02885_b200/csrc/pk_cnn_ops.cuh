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

// Programmatic dependent launch (every launch of a step program after the
// first carries the PDL attribute, pk_cnn.cu launch_k): a block first lets the
// next launch of the chain start — its blocks are placed as SM resources free
// up and park in griddepcontrol.wait — then waits for its predecessor's
// completion and memory flush before it touches global data.  This hides the
// launch + ramp of each of a step's few hundred launches behind the previous
// one's tail.  A block waits unconditionally, so completion stays transitive
// along the chain.  (Without the attribute both instructions are no-ops.)
__device__ __forceinline__ void pdl_gate() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

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
// Row-strided column reductions.  Thread t owns channel group j = t % cgp
// (cgp = pow2 >= c/8, 8 channels = one 16-byte vector) of row lane
// rl = t / cgp, and visits rows r0 + rl, + nr, ... < r1 (nr = 256 / cgp),
// kU rows per round with every load of the round issued before any use (the
// memory-level parallelism these HBM/L2-bound kernels live on).  Per-thread
// sums become the block's partial record in a fixed order (smem transpose, row
// lanes summed in lane order), so a block's record depends only on its rows.
// ------------------------------------------------------------------------------
constexpr int kU = 4;

struct Lanes {
  int cgs, cgp, rl, nr, ch;
  bool on;
};
__device__ __forceinline__ Lanes lanes_of(int c) {
  Lanes L;
  L.cgs = c >> 3;
  L.cgp = 1;
  while (L.cgp < L.cgs) L.cgp <<= 1;
  const int t = threadIdx.x, j = t & (L.cgp - 1);
  L.rl = t / L.cgp;
  L.nr = kBlock / L.cgp;
  L.ch = 8 * j;
  L.on = j < L.cgs;
  return L;
}

__device__ __forceinline__ uint4 ldg16(const uint8_t* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}
__device__ __forceinline__ void unpack8(const uint4& u, float (&v)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float (&v)[8]) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
  return u;
}

// Σ over the block's row lanes of s1 / s2 → out[0..c) / out[c..2c).
__device__ __forceinline__ void block_colsum2(const Lanes& L, int c, const float (&s1)[8],
                                              const float (&s2)[8], float* out) {
  __shared__ __align__(16) float sh[2 * 2048];  // nr * 2c <= 4096
  const int n2 = 2 * c;
  if (L.on) {
    float4* d1 = reinterpret_cast<float4*>(sh + L.rl * n2 + L.ch);
    float4* d2 = reinterpret_cast<float4*>(sh + L.rl * n2 + c + L.ch);
    d1[0] = make_float4(s1[0], s1[1], s1[2], s1[3]);
    d1[1] = make_float4(s1[4], s1[5], s1[6], s1[7]);
    d2[0] = make_float4(s2[0], s2[1], s2[2], s2[3]);
    d2[1] = make_float4(s2[4], s2[5], s2[6], s2[7]);
  }
  __syncthreads();
  for (int o = threadIdx.x; o < n2; o += kBlock) {
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    int l = 0;
    for (; l + 4 <= L.nr; l += 4) {
      a0 += sh[l * n2 + o];
      a1 += sh[(l + 1) * n2 + o];
      a2 += sh[(l + 2) * n2 + o];
      a3 += sh[(l + 3) * n2 + o];
    }
    for (; l < L.nr; ++l) a0 += sh[l * n2 + o];
    out[o] = (a0 + a1) + (a2 + a3);
  }
}

// Row loop of a column reduction over NIN bf16 tensors: base[i] points at the
// thread's channel group of row 0 of tensor i (pitch bytes per row).  fn(v)
// folds row r's NIN vectors into the thread's sums.
template <int NIN, class Fn>
__device__ __forceinline__ void row_loop(const Lanes& L, int r0, int r1,
                                         const uint8_t* const (&base)[NIN],
                                         const size_t (&pitch)[NIN], Fn&& fn) {
  if (!L.on) return;
  int r = r0 + L.rl;
  for (; r + (kU - 1) * L.nr < r1; r += kU * L.nr) {
    uint4 v[kU][NIN];
#pragma unroll
    for (int u = 0; u < kU; ++u)
#pragma unroll
      for (int i = 0; i < NIN; ++i) v[u][i] = ldg16(base[i] + (size_t)(r + u * L.nr) * pitch[i]);
#pragma unroll
    for (int u = 0; u < kU; ++u) fn(v[u], r + u * L.nr);
  }
  for (; r < r1; r += L.nr) {
    uint4 v[NIN];
#pragma unroll
    for (int i = 0; i < NIN; ++i) v[i] = ldg16(base[i] + (size_t)r * pitch[i]);
    fn(v, r);
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
  for (int i = threadIdx.x; i < nout; i += kBlock) {  // the group's records: loads first
    float r[kRedGroup];
#pragma unroll
    for (int b = 0; b < kRedGroup; ++b)
      r[b] = b0 + b < b1 ? __ldcg(ws + (long long)(b0 + b) * stride + i) : 0.f;
    double v = 0.0;
#pragma unroll
    for (int b = 0; b < kRedGroup; ++b)
      if (b0 + b < b1) v += r[b];
    grec[(long long)grp * nout + i] = v;
  }
  if (!ticket(counters, ngroups)) return false;
  for (int i = threadIdx.x; i < nout; i += kBlock) {
    double r[kRedGroup];
#pragma unroll
    for (int g = 0; g < kRedGroup; ++g)
      r[g] = g < ngroups ? __ldcg(grec + (long long)g * nout + i) : 0.0;
    double v = 0.0;
#pragma unroll
    for (int g = 0; g < kRedGroup; ++g)
      if (g < ngroups) v += r[g];
    tot[i] = v;
  }
  __syncthreads();
  return true;
}

// Partial records consumed by the NEXT kernel (BN statistics, BN backward):
// every block writes its fp32 record ws[blk][nout]; when the member has more
// than kRedGroup blocks, the last block of each group (ticket) also folds the
// group's records, in block order, into an fp64 group record.  No second
// ticket level: the consumer (the apply kernel) sums the <= kRedGroup records
// of a column itself, in a fixed order — the same sums tree_reduce forms, one
// dependent global round trip shorter on the producer's critical path.
__device__ __forceinline__ void group_fold(float* ws, int blk, int nblk, int nout, int* counters) {
  if (nblk <= kRedGroup) return;
  const int grp = blk / kRedGroup;
  const int b0 = grp * kRedGroup, b1 = min(nblk, b0 + kRedGroup);
  double* grec = reinterpret_cast<double*>(ws + (((long long)nblk * nout + 1) & ~1LL));
  if (!ticket(counters + 1 + grp, b1 - b0)) return;
  for (int i = threadIdx.x; i < nout; i += kBlock) {
    double v = 0.0;
    for (int b = b0; b < b1; ++b) v += __ldcg(ws + (long long)b * nout + i);
    grec[(long long)grp * nout + i] = v;
  }
}
__device__ __forceinline__ double record_total(const float* ws, int nblk, int nout, int i) {
  // <= kRedGroup records either way; the group records of large members (the
  // bandwidth-bound layers) are all loaded before they are summed in order
  double v = 0.0;
  if (nblk <= kRedGroup) {
    for (int b = 0; b < nblk; ++b) v += __ldcg(ws + (long long)b * nout + i);
  } else {
    const double* grec =
        reinterpret_cast<const double*>(ws + (((long long)nblk * nout + 1) & ~1LL));
    const int ng = (nblk + kRedGroup - 1) / kRedGroup;
    double r[kRedGroup];
#pragma unroll
    for (int g = 0; g < kRedGroup; ++g) r[g] = g < ng ? __ldcg(grec + (long long)g * nout + i) : 0.0;
#pragma unroll
    for (int g = 0; g < kRedGroup; ++g)
      if (g < ng) v += r[g];
  }
  return v;
}

// profiling helper (pk_cnn_prog_profile): keep the stream busy for `cycles`
__global__ void k_spin(long long cycles) {
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
}

// ============================== batch norm =====================================
__global__ void __launch_bounds__(kBlock, 4) k_bn_stats(const __grid_constant__ Pack<pk_cnn_bn> G) {
  pdl_gate();
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_bn& P = G.p[pi];
  const int blk = blockIdx.x - G.blk0[pi], nblk = G.blk0[pi + 1] - G.blk0[pi];
  const int r0 = blk * P.rpb, r1 = min(P.rows, r0 + P.rpb);
  const Lanes L = lanes_of(P.c);
  float s1[8], s2[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) s1[e] = s2[e] = 0.f;
  const uint8_t* const base[1] = {static_cast<const uint8_t*>(P.x) + 2 * L.ch};
  const size_t pitch[1] = {(size_t)P.ldx * 2};
  row_loop<1>(L, r0, r1, base, pitch, [&](const uint4 (&v)[1], int) {
    float a[8];
    unpack8(v[0], a);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      s1[e] += a[e];
      s2[e] = fmaf(a[e], a[e], s2[e]);
    }
  });
  block_colsum2(L, P.c, s1, s2, P.ws + (size_t)blk * 2 * P.c);
  group_fold(P.ws, blk, nblk, 2 * P.c, P.counter);
}

// g = dout · act'(fout); xhat = (x - mean)·rstd; partial sums of g and g·xhat
__global__ void __launch_bounds__(kBlock, 2) k_bn_bwd_reduce(const __grid_constant__ Pack<pk_cnn_bn> G) {
  pdl_gate();
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_bn& P = G.p[pi];
  const int blk = blockIdx.x - G.blk0[pi], nblk = G.blk0[pi + 1] - G.blk0[pi];
  const int r0 = blk * P.rpb, r1 = min(P.rows, r0 + P.rpb);
  const Lanes L = lanes_of(P.c);
  float s1[8], s2[8], mean[8], rs[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) s1[e] = s2[e] = 0.f;
  if (L.on) {
    ld8f(P.stats + L.ch, mean);
    ld8f(P.stats + P.c + L.ch, rs);
  }
  auto fold = [&](const float (&d)[8], const float (&x)[8], const float* fo) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float g = fo ? d[e] * act_bwd(fo[e], P.act) : d[e];
      s1[e] += g;
      s2[e] = fmaf(g, (x[e] - mean[e]) * rs[e], s2[e]);
    }
  };
  if (P.act != PK_CNN_ACT_NONE) {
    const uint8_t* const base[3] = {static_cast<const uint8_t*>(P.dout) + 2 * L.ch,
                                    static_cast<const uint8_t*>(P.x) + 2 * L.ch,
                                    static_cast<const uint8_t*>(P.fout) + 2 * L.ch};
    const size_t pitch[3] = {(size_t)P.ldd * 2, (size_t)P.ldx * 2, (size_t)P.ldo * 2};
    row_loop<3>(L, r0, r1, base, pitch, [&](const uint4 (&v)[3], int) {
      float d[8], x[8], fo[8];
      unpack8(v[0], d);
      unpack8(v[1], x);
      unpack8(v[2], fo);
      fold(d, x, fo);
    });
  } else {
    const uint8_t* const base[2] = {static_cast<const uint8_t*>(P.dout) + 2 * L.ch,
                                    static_cast<const uint8_t*>(P.x) + 2 * L.ch};
    const size_t pitch[2] = {(size_t)P.ldd * 2, (size_t)P.ldx * 2};
    row_loop<2>(L, r0, r1, base, pitch, [&](const uint4 (&v)[2], int) {
      float d[8], x[8];
      unpack8(v[0], d);
      unpack8(v[1], x);
      fold(d, x, nullptr);
    });
  }
  block_colsum2(L, P.c, s1, s2, P.ws + (size_t)blk * 2 * P.c);
  group_fold(P.ws, blk, nblk, 2 * P.c, P.counter);
}

// ------------------------------------------------------------------------------
// BN apply kernels: a block owns a tile of rows [r0, r0 + R) x channel groups
// [g0, g0 + gw) (gw <= kApplyGroups), R = kApplyItems / min(cgs, kApplyGroups);
// its per-channel coefficients are computed once into shared memory, then each
// thread handles items t, t + 256, ... (kU of them, loads issued together).
// ------------------------------------------------------------------------------
constexpr int kApplyGroups = 32, kApplyItems = kU * kBlock;

struct ApplyTile {
  int r0, r1, R, g0, gw;  // the block's rows [r0, r1) in steps of R rows
};
constexpr int kApplyMaxBlocks = 4 * 148;  // per problem; larger layers loop over row tiles
__host__ __device__ __forceinline__ int apply_groups(int c) {
  return (c >> 3) < kApplyGroups ? (c >> 3) : kApplyGroups;
}
// row tiles per block of a problem: spans of rt row tiles (elementwise kernels:
// any partition gives the same result)
// maxb: block budget of the problem (pk_cnn_bn.pad0, set per launch by the host
// from the number of problems sharing it; 0 = kApplyMaxBlocks)
__host__ __device__ __forceinline__ void apply_shape(int rows, int c, int maxb, int& ncg, int& nrt,
                                                     int& rt) {
  const int cgs = c >> 3, G = apply_groups(c), R = kApplyItems / G;
  ncg = (cgs + G - 1) / G;
  nrt = (rows + R - 1) / R;
  const int spans = max(1, (maxb > 0 ? maxb : kApplyMaxBlocks) / ncg);
  rt = (nrt + spans - 1) / spans;
}
__host__ __device__ __forceinline__ int apply_blocks(int rows, int c, int maxb) {
  int ncg, nrt, rt;
  apply_shape(rows, c, maxb, ncg, nrt, rt);
  return ((nrt + rt - 1) / rt) * ncg;
}
__device__ __forceinline__ ApplyTile apply_tile(int b, int rows, int c, int maxb) {
  const int cgs = c >> 3, G = apply_groups(c);
  int ncg, nrt, rt;
  apply_shape(rows, c, maxb, ncg, nrt, rt);
  ApplyTile T;
  T.R = kApplyItems / G;
  const int tr = b / ncg, tg = b - tr * ncg;
  T.r0 = tr * rt * T.R;
  T.r1 = min(rows, T.r0 + rt * T.R);
  T.g0 = tg * G;
  T.gw = min(G, cgs - T.g0);
  return T;
}

__global__ void __launch_bounds__(kBlock, 3) k_bn_apply(const __grid_constant__ Pack<pk_cnn_bn> G) {
  pdl_gate();
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_bn& P = G.p[pi];
  const ApplyTile T = apply_tile(blockIdx.x - G.blk0[pi], P.rows, P.c, P.pad0);
  __shared__ float scale[kApplyGroups * 8], shift[kApplyGroups * 8];
  const int t = threadIdx.x;
  if (t < T.gw * 8) {  // y = x·(γ·rstd) + (β − mean·γ·rstd)
    const int ch = T.g0 * 8 + t;
    float mean, rs;
    if (P.use_running) {
      mean = P.run_mean[ch];
      rs = (float)(1.0 / sqrt((double)P.run_var[ch] + (double)P.eps));
    } else {
      // batch statistics from k_bn_stats' partial records; the tiles of row
      // block 0 publish them (and the running statistics) exactly once
      const int nblk = (P.rows + P.rpb - 1) / P.rpb;
      const double dm = record_total(P.ws, nblk, 2 * P.c, ch) / P.rows;
      const double var = fmax(record_total(P.ws, nblk, 2 * P.c, P.c + ch) / P.rows - dm * dm, 0.0);
      mean = (float)dm;
      rs = (float)(1.0 / sqrt(var + (double)P.eps));
      if (T.r0 == 0) {
        P.stats[ch] = mean;
        P.stats[P.c + ch] = rs;
        if (P.run_mean) {
          const double unb = P.rows > 1 ? var * P.rows / (P.rows - 1) : var;
          P.run_mean[ch] = (float)((1.0 - P.momentum) * P.run_mean[ch] + P.momentum * dm);
          P.run_var[ch] = (float)((1.0 - P.momentum) * P.run_var[ch] + P.momentum * unb);
        }
      }
    }
    const float g = P.gamma[ch] * rs;
    scale[t] = g;
    shift[t] = P.beta[ch] - mean * g;
  }
  __syncthreads();
  const int nitems = T.R * T.gw;
  for (int rb = T.r0; rb < T.r1; rb += T.R) {
  int row[kU], cg[kU];
  uint4 x[kU], rv[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    const int i = t + u * kBlock, rr = i / T.gw;
    row[u] = rb + rr;
    cg[u] = i - rr * T.gw;
    if (i < nitems && row[u] < T.r1) {
      const int ch = (T.g0 + cg[u]) * 8;
      x[u] = ldg16(bptr(P.x, row[u], P.ldx, ch));
      if (P.res) rv[u] = ldg16(bptr(P.res, row[u], P.ldr, ch));
    } else {
      row[u] = -1;
    }
  }
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    if (row[u] < 0) continue;
    float v[8], r[8];
    unpack8(x[u], v);
    if (P.res) unpack8(rv[u], r);
    const float* sc = scale + 8 * cg[u];
    const float* sf = shift + 8 * cg[u];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      float y = fmaf(v[e], sc[e], sf[e]);
      if (P.res) y += r[e];
      v[e] = act_fwd(y, P.act);
    }
    *reinterpret_cast<uint4*>(bptr(P.out, row[u], P.ldo, (T.g0 + cg[u]) * 8)) = pack8(v);
  }
  }
}

template <bool ACT, bool SIDE>
__device__ __forceinline__ void bn_bwd_apply_impl(const Pack<pk_cnn_bn>& G) {
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_bn& P = G.p[pi];
  const ApplyTile T = apply_tile(blockIdx.x - G.blk0[pi], P.rows, P.c, P.pad0);
  // dx = γ·rstd·(g − mean(g) − xhat·mean(g·xhat)) = ca·g + cb·x + cc per channel
  __shared__ float cas[kApplyGroups * 8], cbs[kApplyGroups * 8], ccs[kApplyGroups * 8];
  const int t = threadIdx.x;
  if (t < T.gw * 8) {
    const int ch = T.g0 * 8 + t;
    const float mean = P.stats[ch], rs = P.stats[P.c + ch];
    // Σg and Σg·xhat from k_bn_bwd_reduce's partial records; the tiles of row
    // block 0 publish dβ / dγ (and the non-finite flag) exactly once
    const int nblk = (P.rows + P.rpb - 1) / P.rpb;
    const double t1 = record_total(P.ws, nblk, 2 * P.c, ch);
    const double t2 = record_total(P.ws, nblk, 2 * P.c, P.c + ch);
    const float mg = (float)(t1 / P.rows), mgx = (float)(t2 / P.rows);
    if (T.r0 == 0) {
      P.dbeta[ch] = (float)t1;
      P.dgamma[ch] = (float)t2;
      if (!isfinite(t1) || !isfinite(t2)) *P.flag = 1;
    }
    const float ca = P.gamma[ch] * rs, cb = -ca * rs * mgx;
    cas[t] = ca;
    cbs[t] = cb;
    ccs[t] = -ca * mg - cb * mean;
  }
  __syncthreads();
  constexpr bool act = ACT;
  const int nitems = T.R * T.gw;
  for (int rb = T.r0; rb < T.r1; rb += T.R) {
  int row[kU], cg[kU];
  uint4 d[kU], x[kU], fo[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    const int i = t + u * kBlock, rr = i / T.gw;
    row[u] = rb + rr;
    cg[u] = i - rr * T.gw;
    if (i < nitems && row[u] < T.r1) {
      const int ch = (T.g0 + cg[u]) * 8;
      d[u] = ldg16(bptr(P.dout, row[u], P.ldd, ch));
      x[u] = ldg16(bptr(P.x, row[u], P.ldx, ch));
      if (act) fo[u] = ldg16(bptr(P.fout, row[u], P.ldo, ch));
    } else {
      row[u] = -1;
    }
  }
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    if (row[u] < 0) continue;
    const int ch = (T.g0 + cg[u]) * 8;
    float g[8], xv[8], f[8], dx[8];
    unpack8(d[u], g);
    unpack8(x[u], xv);
    if (act) unpack8(fo[u], f);
    const float* ca = cas + 8 * cg[u];
    const float* cb = cbs + 8 * cg[u];
    const float* cc = ccs + 8 * cg[u];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      if (act) g[e] *= act_bwd(f[e], P.act);
      dx[e] = fmaf(ca[e], g[e], fmaf(cb[e], xv[e], cc[e]));
    }
    uint8_t* pdx = bptr(P.dx, row[u], P.ldx2, ch);
    if (SIDE && P.accumulate) {
      float o[8];
      ld8(pdx, o);
#pragma unroll
      for (int e = 0; e < 8; ++e) dx[e] += o[e];
    }
    *reinterpret_cast<uint4*>(pdx) = pack8(dx);
    if (SIDE && P.dres) {
      uint8_t* pr = bptr(P.dres, row[u], P.ldr, ch);
      if (P.res_accumulate) {
        float o[8];
        ld8(pr, o);
#pragma unroll
        for (int e = 0; e < 8; ++e) g[e] += o[e];
      }
      *reinterpret_cast<uint4*>(pr) = pack8(g);
    }
  }
  }
}

// specialised on the activation and on the side outputs (accumulated dX, the
// residual gradient): the plain form needs fewer registers (3 blocks / SM)
template <bool ACT, bool SIDE>
__global__ void __launch_bounds__(kBlock, (SIDE || ACT) ? 2 : 3) k_bn_bwd_apply_t(const __grid_constant__ Pack<pk_cnn_bn> G) {
  pdl_gate();
  bn_bwd_apply_impl<ACT, SIDE>(G);
}

// ============================ depthwise conv =====================================
// generic shapes: one thread per (output pixel, channel group)
__device__ __forceinline__ void dw_fprop_items(const pk_cnn_dw& P, int blk) {
  const int cgs = P.c >> 3;
  const long long item = (long long)blk * kBlock + threadIdx.x;
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

__device__ __forceinline__ void dw_dgrad_items(const pk_cnn_dw& P, int blk) {
  const int cgs = P.c >> 3;
  const long long item = (long long)blk * kBlock + threadIdx.x;
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
__device__ __forceinline__ void dw_wgrad_generic(const pk_cnn_dw& P, int blk, int nblk) {
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

// ------------------------------------------------------------------------------
// 3x3 depthwise fast paths.
//   FPROP / DGRAD: one thread per (pixel, channel group) of the output plane, all
//     nine source vectors and nine weight vectors loaded before any FMA, 32-bit
//     index math (the generic path below walks taps with data-dependent skips).
//   WGRAD: a block owns one CHUNK of <= 8 channel groups (64 channels) and one
//     split of the member's output pixels; thread = (channel group j, kernel
//     row r, pixel lane), kU pixels' loads (dy + the row's three x vectors)
//     issued before their FMAs, 24 accumulators per thread.  The block's
//     [9][64] record is summed over its lanes in lane order; a member's
//     splits of a chunk (nchunk x nsplit <= 256 blocks) are folded in split
//     order (fp64, tree_reduce: groups of 16, loads issued before the adds).
//     Small records instead of [9][c] records per block (a 1x1x480 layer:
//     44 -> 12 us).
// ------------------------------------------------------------------------------
__host__ __device__ __forceinline__ bool dw_fast(const pk_cnn_dw& P, int mode) {
  (void)mode;
  return P.r == 3 && P.s == 3 && (P.stride == 1 || P.stride == 2);
}
// WGRAD channel groups per block (a chunk), chunks per member, pixel lanes of
// a 256-thread block ((256 / groups) / 3 kernel-row triples), splits per chunk
constexpr int kDwChunkGroups = 8;
__host__ __device__ __forceinline__ int dw_wgrad_cgb(int c) {
  int g = 1;
  while (g < (c >> 3)) g <<= 1;
  return g < kDwChunkGroups ? g : kDwChunkGroups;
}
__host__ __device__ __forceinline__ int dw_wgrad_chunks(int c) {
  const int b = dw_wgrad_cgb(c);
  return ((c >> 3) + b - 1) / b;
}
__host__ __device__ __forceinline__ int dw_wgrad_lanes(int c) { return (256 / dw_wgrad_cgb(c)) / 3; }

template <int MODE, int ST>
__device__ __forceinline__ void dw_items3(const pk_cnn_dw& P, int blk) {
  const int cgs = P.c >> 3;
  const int oh = MODE == PK_CNN_DW_DGRAD ? P.h : P.p, ow = MODE == PK_CNN_DW_DGRAD ? P.w : P.q;
  const int item = blk * kBlock + (int)threadIdx.x;
  if (item >= P.n * oh * ow * cgs) return;
  const int m = item / cgs, ch = 8 * (item - m * cgs);
  const int n = m / (oh * ow), rem = m - n * (oh * ow);
  const int y = rem / ow, x = rem - y * ow;
  const uint8_t* src = static_cast<const uint8_t*>(MODE == PK_CNN_DW_DGRAD ? P.dy : P.x) + 2 * ch;
  const int sh = MODE == PK_CNN_DW_DGRAD ? P.p : P.h, sw = MODE == PK_CNN_DW_DGRAD ? P.q : P.w;
  const size_t pitch = (size_t)(MODE == PK_CNN_DW_DGRAD ? P.ldy : P.ldx) * 2;
  uint4 v[9], wv[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      int sy, sx;
      bool ok;
      if (MODE == PK_CNN_DW_DGRAD) {  // dx(y,x) += dy((y+pad-r)/st, (x+pad-s)/st)·w[r][s]
        const int ty = y + P.pad - r, tx = x + P.pad - s;
        sy = ST == 1 ? ty : ty >> 1;
        sx = ST == 1 ? tx : tx >> 1;
        ok = ty >= 0 && tx >= 0 && (ST == 1 || ((ty | tx) & 1) == 0) && sy < sh && sx < sw;
      } else {
        sy = y * ST - P.pad + r;
        sx = x * ST - P.pad + s;
        ok = (unsigned)sy < (unsigned)sh && (unsigned)sx < (unsigned)sw;
      }
      v[3 * r + s] = ok ? ldg16(src + ((size_t)(n * sh + sy) * sw + sx) * pitch)
                        : make_uint4(0, 0, 0, 0);
      wv[3 * r + s] = ldg16(bptr(P.wt, 3 * r + s, P.c, ch));
    }
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
#pragma unroll
  for (int k = 0; k < 9; ++k) {  // taps in (r, s) order, as the generic path
    float a[8], w[8];
    unpack8(v[k], a);
    unpack8(wv[k], w);
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = fmaf(a[e], w[e], acc[e]);
  }
  const int old = MODE == PK_CNN_DW_DGRAD ? P.ldx : P.ldy;
  *reinterpret_cast<uint4*>(bptr(P.y, m, old, ch)) = pack8(acc);
}

// 3x3 pad-1 FPROP / DGRAD on output strips: a thread computes XS consecutive
// outputs of one row for one channel group, so the source vectors the strip's
// windows share are loaded once (stride 1: 3 x (XS+2) sources for XS outputs,
// 6.75 loads per output with the weights instead of 18).  Stride-2 DGRAD
// visits only the taps whose stride quotient is exact (x0 even: tap s of
// output i is live iff i + 1 - s is even).  Taps accumulate in (r, s) order
// per output, as in dw_items3.
__host__ __device__ __forceinline__ bool dw_strip_ok(const pk_cnn_dw& P) {
  return P.r == 3 && P.s == 3 && P.pad == 1 && (P.stride == 1 || P.stride == 2);
}
__host__ __device__ __forceinline__ int dw_strip_xs(int mode, int stride) {
  return (mode == PK_CNN_DW_FPROP && stride == 2) ? 2 : 4;
}
template <int MODE, int ST>
__device__ __forceinline__ void dw_strip(const pk_cnn_dw& P, int blk) {
  constexpr int XS = (MODE == PK_CNN_DW_FPROP && ST == 2) ? 2 : 4;
  constexpr bool D2 = MODE == PK_CNN_DW_DGRAD && ST == 2;
  // source columns of a strip: FPROP (x0·ST − 1) + [0, (XS−1)·ST + 3); DGRAD
  // stride 1: (x0 − 1) + [0, XS + 2); DGRAD stride 2: x0/2 + [0, 3)
  constexpr int NC = D2 ? 3 : (MODE == PK_CNN_DW_FPROP ? (XS - 1) * ST + 3 : XS + 2);
  const int cgs = P.c >> 3;
  const int oh = MODE == PK_CNN_DW_DGRAD ? P.h : P.p, ow = MODE == PK_CNN_DW_DGRAD ? P.w : P.q;
  const int ns = (ow + XS - 1) / XS;
  const int item = blk * kBlock + (int)threadIdx.x;
  if (item >= P.n * oh * ns * cgs) return;
  const int cgi = item % cgs;
  int rest = item / cgs;
  const int sp = rest % ns;
  rest /= ns;
  const int y = rest % oh, n = rest / oh;
  const int x0 = sp * XS, ch = 8 * cgi;
  const uint8_t* src = static_cast<const uint8_t*>(MODE == PK_CNN_DW_DGRAD ? P.dy : P.x) + 2 * ch;
  const int sh = MODE == PK_CNN_DW_DGRAD ? P.p : P.h, sw = MODE == PK_CNN_DW_DGRAD ? P.q : P.w;
  const size_t pitch = (size_t)(MODE == PK_CNN_DW_DGRAD ? P.ldy : P.ldx) * 2;
  const int c0 = D2 ? (x0 >> 1) : (MODE == PK_CNN_DW_FPROP ? x0 * ST - 1 : x0 - 1);
  uint4 v[3][NC], wv[9];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    int sy;
    bool rok;
    if (MODE == PK_CNN_DW_FPROP) {
      sy = y * ST - 1 + r;
      rok = (unsigned)sy < (unsigned)sh;
    } else if (!D2) {
      sy = y + 1 - r;
      rok = (unsigned)sy < (unsigned)sh;
    } else {
      const int ty = y + 1 - r;
      sy = ty >> 1;
      rok = ty >= 0 && !(ty & 1) && sy < sh;
    }
    const uint8_t* row = src + (size_t)(n * sh + sy) * sw * pitch;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int sx = c0 + k;
      v[r][k] = rok && (unsigned)sx < (unsigned)sw ? ldg16(row + (size_t)sx * pitch)
                                                  : make_uint4(0, 0, 0, 0);
    }
  }
#pragma unroll
  for (int k = 0; k < 9; ++k) wv[k] = ldg16(bptr(P.wt, k, P.c, ch));
  float acc[XS][8];
#pragma unroll
  for (int i = 0; i < XS; ++i)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[i][e] = 0.f;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      float w[8];
      unpack8(wv[3 * r + s], w);
#pragma unroll
      for (int i = 0; i < XS; ++i) {
        int k;
        if (MODE == PK_CNN_DW_FPROP) k = i * ST + s;
        else if (!D2) k = i + 2 - s;
        else {
          if ((i + 1 - s) & 1) continue;  // not an exact stride quotient
          k = (i + 1 - s) >> 1;
        }
        float a[8];
        unpack8(v[r][k], a);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[i][e] = fmaf(a[e], w[e], acc[i][e]);
      }
    }
  const int old = MODE == PK_CNN_DW_DGRAD ? P.ldx : P.ldy;
#pragma unroll
  for (int i = 0; i < XS; ++i)
    if (x0 + i < ow)
      *reinterpret_cast<uint4*>(bptr(P.y, (long long)(n * oh + y) * ow + x0 + i, old, ch)) =
          pack8(acc[i]);
}

__device__ __forceinline__ void dw_fast_wgrad(const pk_cnn_dw& P, int blk) {
  const int cgb = dw_wgrad_cgb(P.c), CC = 8 * cgb, n9 = 9 * CC;
  const int pq = P.p * P.q, M = P.n * pq;
  const int nsplit = (M + P.ppb - 1) / P.ppb;
  const int chunk = blk / nsplit, split = blk - chunk * nsplit;
  const int t = threadIdx.x, j = t % cgb, rest = t / cgb;
  const int lanes = dw_wgrad_lanes(P.c);
  const int r = rest % 3, rl = rest / 3, ch = 8 * (chunk * cgb + j);
  const bool on = ch < P.c && rl < lanes;
  float acc[3][8];
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[k][e] = 0.f;
  if (on) {
    const uint8_t* xb = static_cast<const uint8_t*>(P.x) + 2 * ch;
    const uint8_t* dyb = static_cast<const uint8_t*>(P.dy) + 2 * ch;
    const size_t xp = (size_t)P.ldx * 2, dp = (size_t)P.ldy * 2;
    const int m1 = min(M, (split + 1) * P.ppb);
    // one pixel: dy vector + the three x vectors of kernel row r
    auto load = [&](int m, uint4& d, uint4 (&xv)[3]) {
      const int n = m / pq, rem = m - n * pq, oy = rem / P.q, ox = rem - oy * P.q;
      d = ldg16(dyb + (size_t)m * dp);
      const int iy = oy * P.stride - P.pad + r, ix0 = ox * P.stride - P.pad;
      const bool rok = (unsigned)iy < (unsigned)P.h;
      const uint8_t* xr = xb + (size_t)(n * P.h + iy) * P.w * xp;
#pragma unroll
      for (int s = 0; s < 3; ++s)
        xv[s] = rok && (unsigned)(ix0 + s) < (unsigned)P.w ? ldg16(xr + (size_t)(ix0 + s) * xp)
                                                          : make_uint4(0, 0, 0, 0);
    };
    auto fold = [&](const uint4& d, const uint4 (&xv)[3]) {
      float dv[8];
      unpack8(d, dv);
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        float a[8];
        unpack8(xv[s], a);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[s][e] = fmaf(dv[e], a[e], acc[s][e]);
      }
    };
    int m = split * P.ppb + rl;
    for (; m + (kU - 1) * lanes < m1; m += kU * lanes) {  // kU pixels' loads, then math
      uint4 d[kU], xv[kU][3];
#pragma unroll
      for (int u = 0; u < kU; ++u) load(m + u * lanes, d[u], xv[u]);
#pragma unroll
      for (int u = 0; u < kU; ++u) fold(d[u], xv[u]);
    }
    for (; m < m1; m += lanes) {
      uint4 d, xv[3];
      load(m, d, xv);
      fold(d, xv);
    }
  }
  // block record [tap][CC]: thread (j, r, rl) holds taps 3r .. 3r+2 of its 8 channels
  __shared__ __align__(16) float sh[6144];  // lanes * 9 * CC <= (256 / cgb / 3) * 72 cgb
  if (rl < lanes) {
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      float4* dst = reinterpret_cast<float4*>(sh + rl * n9 + (3 * r + s) * CC + 8 * j);
      dst[0] = make_float4(acc[s][0], acc[s][1], acc[s][2], acc[s][3]);
      dst[1] = make_float4(acc[s][4], acc[s][5], acc[s][6], acc[s][7]);
    }
  }
  __syncthreads();
  const int c0 = chunk * CC;
  auto out_index = [&](int o, int& di) {  // record slot -> dw[tap][c] (false: padding)
    const int tap = o / CC, cc = o - tap * CC;
    di = tap * P.c + c0 + cc;
    return c0 + cc < P.c;
  };
  bool bad = false;
  if (nsplit == 1) {  // the chunk's only block: its record is the gradient
    for (int o = t; o < n9; o += kBlock) {
      float a = 0.f;
      for (int l = 0; l < lanes; ++l) a += sh[l * n9 + o];
      int di;
      if (out_index(o, di)) {
        P.dw[di] = a;
        bad |= !isfinite(a);
      }
    }
    if (bad) *P.flag = 1;
    return;
  }
  // a chunk's records and tree_reduce workspace: [nsplit][n9] floats, fp64 group
  // records, totals (cnn.py _red_ws(n9, nsplit, n9) floats per chunk)
  const long long cstride = (((long long)nsplit * n9 + 1) & ~1LL) +
                            2LL * n9 * ((nsplit + kRedGroup - 1) / kRedGroup + 1) + 2;
  float* cws = P.ws + chunk * cstride;
  float* rec = cws + (long long)split * n9;
  for (int o = t; o < n9; o += kBlock) {
    float a = 0.f;
    for (int l = 0; l < lanes; ++l) a += sh[l * n9 + o];
    rec[o] = a;
  }
  double* tot;
  if (!tree_reduce(cws, split, nsplit, n9, n9, P.counter + (kRedGroup + 1) * chunk, &tot)) return;
  for (int o = t; o < n9; o += kBlock) {
    int di;
    if (out_index(o, di)) {
      P.dw[di] = (float)tot[o];
      bad |= !isfinite(tot[o]);
    }
  }
  if (bad) *P.flag = 1;
}

__global__ void __launch_bounds__(kBlock) k_dw_fprop(const __grid_constant__ Pack<pk_cnn_dw> G) {
  pdl_gate();
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_dw& P = G.p[pi];
  const int blk = blockIdx.x - G.blk0[pi];
  if (dw_strip_ok(P)) {
    if (P.stride == 1) dw_strip<PK_CNN_DW_FPROP, 1>(P, blk);
    else dw_strip<PK_CNN_DW_FPROP, 2>(P, blk);
  } else if (dw_fast(P, PK_CNN_DW_FPROP)) {
    if (P.stride == 1) dw_items3<PK_CNN_DW_FPROP, 1>(P, blk);
    else dw_items3<PK_CNN_DW_FPROP, 2>(P, blk);
  }
  else dw_fprop_items(P, blk);
}

__global__ void __launch_bounds__(kBlock) k_dw_dgrad(const __grid_constant__ Pack<pk_cnn_dw> G) {
  pdl_gate();
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_dw& P = G.p[pi];
  const int blk = blockIdx.x - G.blk0[pi];
  if (dw_strip_ok(P)) {
    if (P.stride == 1) dw_strip<PK_CNN_DW_DGRAD, 1>(P, blk);
    else dw_strip<PK_CNN_DW_DGRAD, 2>(P, blk);
  } else if (dw_fast(P, PK_CNN_DW_DGRAD)) {
    if (P.stride == 1) dw_items3<PK_CNN_DW_DGRAD, 1>(P, blk);
    else dw_items3<PK_CNN_DW_DGRAD, 2>(P, blk);
  }
  else dw_dgrad_items(P, blk);
}

__global__ void __launch_bounds__(kBlock, 2) k_dw_wgrad(const __grid_constant__ Pack<pk_cnn_dw> G) {
  pdl_gate();
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_dw& P = G.p[pi];
  const int blk = blockIdx.x - G.blk0[pi], nblk = G.blk0[pi + 1] - G.blk0[pi];
  if (dw_fast(P, PK_CNN_DW_WGRAD)) dw_fast_wgrad(P, blk);
  else dw_wgrad_generic(P, blk, nblk);
}

// ================================ pooling ========================================
// Bodies are templates on the window / stride (0 = runtime value) so the
// common shapes (3x3/2 ResNet stem, 2x2/2 LeNet) unroll their tap loops.
template <int R_, int S_, int ST_>
__device__ __forceinline__ void maxpool_fwd_item(const pk_cnn_pool& P, int m, int ch) {
  const int R = R_ ? R_ : P.r, S = S_ ? S_ : P.s, ST = ST_ ? ST_ : P.stride;
  const int n = m / (P.p * P.q), rem = m - n * P.p * P.q;
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
__device__ __forceinline__ void pool_bwd_item(const pk_cnn_pool& P, int m, int ch) {
  const int R = R_ ? R_ : P.r, S = S_ ? S_ : P.s, ST = ST_ ? ST_ : P.stride;
  const int n = m / (P.h * P.w), rem = m - n * P.h * P.w;
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

// Square-window max pooling with a compile-time window / stride: every tap's
// source vector (forward) or every window's dY / argmax pair (backward: an
// input pixel lies in <= ceil(R/ST)^2 windows, rr ≡ iy + pad mod ST) is loaded
// before any is used; the taps / windows are then visited in the (r, s) order
// of maxpool_fwd_item / pool_bwd_item, so the results are the same.
template <int R, int ST>
__device__ __forceinline__ void maxpool_fwd_fast(const pk_cnn_pool& P, int m, int ch) {
  const int n = m / (P.p * P.q), rem = m - n * (P.p * P.q);
  const int oy = rem / P.q, ox = rem - oy * P.q;
  uint4 v[R][R];
  bool ok[R][R];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const int iy = oy * ST - P.pad + r, ix = ox * ST - P.pad + s;
      ok[r][s] = (unsigned)iy < (unsigned)P.h && (unsigned)ix < (unsigned)P.w;
      v[r][s] = ok[r][s] ? ldg16(bptr(P.x, ((long long)n * P.h + iy) * P.w + ix, P.ldx, ch))
                         : make_uint4(0, 0, 0, 0);
    }
  float best[8];
  uint8_t arg[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    best[e] = -INFINITY;
    arg[e] = 0;
  }
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int s = 0; s < R; ++s) {
      if (!ok[r][s]) continue;
      float x[8];
      unpack8(v[r][s], x);
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (x[e] > best[e]) {
          best[e] = x[e];
          arg[e] = (uint8_t)(r * R + s);
        }
    }
  st8(bptr(P.y, m, P.ldy, ch), best);
  uint2 a;
  a.x = arg[0] | (arg[1] << 8) | (arg[2] << 16) | ((uint32_t)arg[3] << 24);
  a.y = arg[4] | (arg[5] << 8) | (arg[6] << 16) | ((uint32_t)arg[7] << 24);
  *reinterpret_cast<uint2*>(P.arg + m * P.c + ch) = a;
}

template <int R, int ST>
__device__ __forceinline__ void maxpool_bwd_fast(const pk_cnn_pool& P, int m, int ch) {
  constexpr int NW = (R + ST - 1) / ST;  // candidate windows per axis
  const int n = m / (P.h * P.w), rem = m - n * (P.h * P.w);
  const int iy = rem / P.w, ix = rem - iy * P.w;
  const int ry = (iy + P.pad) % ST, rx = (ix + P.pad) % ST;
  uint4 d[NW][NW];
  uint2 a[NW][NW];
  bool ok[NW][NW];
#pragma unroll
  for (int j = 0; j < NW; ++j)
#pragma unroll
    for (int k = 0; k < NW; ++k) {
      const int rr = ry + j * ST, ss = rx + k * ST;
      const int ty = iy + P.pad - rr, tx = ix + P.pad - ss;
      ok[j][k] = rr < R && ss < R && ty >= 0 && tx >= 0 && ty / ST < P.p && tx / ST < P.q;
      if (ok[j][k]) {
        const long long o = ((long long)n * P.p + ty / ST) * P.q + tx / ST;
        d[j][k] = ldg16(bptr(P.dy, o, P.ldy, ch));
        a[j][k] = __ldg(reinterpret_cast<const uint2*>(P.arg + o * P.c + ch));
      }
    }
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
#pragma unroll
  for (int j = 0; j < NW; ++j)
#pragma unroll
    for (int k = 0; k < NW; ++k) {
      if (!ok[j][k]) continue;
      float dv[8];
      unpack8(d[j][k], dv);
      const uint8_t* ab = reinterpret_cast<const uint8_t*>(&a[j][k]);
      const int tap = (ry + j * ST) * R + rx + k * ST;
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (ab[e] == tap) acc[e] += dv[e];
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
  pdl_gate();
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_pool& P = G.p[pi];
  const int cgs = P.c >> 3;
  const int item = (blockIdx.x - G.blk0[pi]) * kBlock + threadIdx.x;  // < 2^31 (host check)
  if (item >= P.n * P.p * P.q * cgs) return;
  const int m = item / cgs;
  const int ch = 8 * (item - m * cgs);
  if (P.r == 3 && P.s == 3 && P.stride == 2) maxpool_fwd_fast<3, 2>(P, m, ch);
  else if (P.r == 2 && P.s == 2 && P.stride == 2) maxpool_fwd_fast<2, 2>(P, m, ch);
  else maxpool_fwd_item<0, 0, 0>(P, m, ch);
}

__global__ void __launch_bounds__(kBlock) k_maxpool_bwd(const __grid_constant__ Pack<pk_cnn_pool> G) {
  pdl_gate();
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_pool& P = G.p[pi];
  const int cgs = P.c >> 3;
  const int item = (blockIdx.x - G.blk0[pi]) * kBlock + threadIdx.x;  // < 2^31 (host check)
  if (item >= P.n * P.h * P.w * cgs) return;
  const int m = item / cgs;
  const int ch = 8 * (item - m * cgs);
  if (P.r == 3 && P.s == 3 && P.stride == 2) maxpool_bwd_fast<3, 2>(P, m, ch);
  else if (P.r == 2 && P.s == 2 && P.stride == 2) maxpool_bwd_fast<2, 2>(P, m, ch);
  else pool_bwd_item<0, 0, 0, false>(P, m, ch);
}

// average pool; the global case (window = the whole map) splits each output's
// window over kPoolLanes threads and combines them with a fixed xor tree — for
// maps of >= 16 pixels; smaller maps (CIFAR nets end at 1x1 / 2x2) use one thread
constexpr int kPoolLanes = 8;
__host__ __device__ __forceinline__ int avgpool_lanes(int hw) { return hw >= 16 ? kPoolLanes : 1; }
__global__ void __launch_bounds__(kBlock) k_avgpool_fwd(const __grid_constant__ Pack<pk_cnn_pool> G) {
  pdl_gate();
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_pool& P = G.p[pi];
  const int cgs = P.c >> 3;
  const bool global = P.r == P.h && P.s == P.w && P.pad == 0 && P.p == 1 && P.q == 1;
  const int lanes = global ? avgpool_lanes(P.h * P.w) : 1;
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
    if (lanes > 1) {  // uniform per problem (a block never mixes problems)
#pragma unroll
      for (int o = kPoolLanes / 2; o; o >>= 1)
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
    }
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
  pdl_gate();
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_pool& P = G.p[pi];
  const int cgs = P.c >> 3;
  const int item = (blockIdx.x - G.blk0[pi]) * kBlock + threadIdx.x;  // < 2^31 (host check)
  if (item >= P.n * P.h * P.w * cgs) return;
  const int m = item / cgs;
  const int ch = 8 * (item - m * cgs);
  if (P.r == 2 && P.s == 2 && P.stride == 2) pool_bwd_item<2, 2, 2, true>(P, m, ch);
  else pool_bwd_item<0, 0, 0, true>(P, m, ch);
}

// ======================== softmax cross-entropy head ============================
// one block per member; reference engine.py:211-230 (loss) and :252-264 (dlogits)
__global__ void __launch_bounds__(kBlock) k_xent(const __grid_constant__ Pack<pk_cnn_head> G) {
  pdl_gate();
  const pk_cnn_head& P = G.p[blockIdx.x];
  extern __shared__ float xs[];
  float* rmax = xs;
  float* rsum = xs + P.rows;
  float* rloss = xs + 2 * P.rows;
  int* rlab = reinterpret_cast<int*>(xs + 3 * P.rows);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float inv = 1.f / (float)P.rows;
  if (P.classes <= 32) {
    // narrow heads (CIFAR's 10 classes): a thread per row, every row's logits and
    // label loaded at once (one round trip, not four per row in a warp's
    // sequence); dbias from fixed-order xor-tree sums over each warp's 32 rows
    float* part = xs + 4 * P.rows;  // [ceil(rows / 32)][classes <= 32] warp partials
    const int nrw = (P.rows + 31) / 32;
    for (int r0 = 0; r0 < P.rows; r0 += kBlock) {
      const int r = r0 + threadIdx.x;
      const bool on = r < P.rows;
      const float* z = P.logits + (long long)(on ? r : 0) * P.ldl;
      float zv[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) zv[j] = on && j < P.classes ? z[j] : -INFINITY;
      const int lab = on ? (int)P.labels[P.idx ? P.idx[r] : r] : 0;
      float mx = -INFINITY;
#pragma unroll
      for (int j = 0; j < 32; ++j) mx = fmaxf(mx, zv[j]);
      float se = 0.f, zl = 0.f;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (j < P.classes) se += expf(zv[j] - mx);
        zl = j == lab ? zv[j] : zl;
      }
      if (on) rloss[r] = logf(se) - (zl - mx);
      const float is = 1.f / se;
      if (on && P.dlogits) {
        __nv_bfloat16* d = static_cast<__nv_bfloat16*>(P.dlogits) + (long long)r * P.ldl;
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < P.classes) d[j] = __float2bfloat16_rn((expf(zv[j] - mx) * is - (j == lab ? 1.f : 0.f)) * inv);
        for (int j = P.classes; j < P.ldl; ++j) d[j] = __float2bfloat16_rn(0.f);
      }
      if (P.dbias) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (j >= P.classes) break;
          float g = on ? (expf(zv[j] - mx) / se - (j == lab ? 1.f : 0.f)) * inv : 0.f;
#pragma unroll
          for (int o = 16; o; o >>= 1) g += __shfl_xor_sync(0xffffffffu, g, o);
          if (lane == 0 && r0 + warp * 32 < P.rows) part[(r0 / 32 + warp) * P.classes + j] = g;
        }
      }
    }
    __syncthreads();
    bool bad = false;
    if (P.dbias) {
      for (int j = threadIdx.x; j < P.classes; j += kBlock) {
        float s = 0.f;
        for (int w = 0; w < nrw; ++w) s += part[w * P.classes + j];
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
    return;
  }
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
__global__ void __launch_bounds__(kBlock, 2) k_bias_act_bwd(const __grid_constant__ Pack<pk_cnn_bias> G) {
  pdl_gate();
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_bias& P = G.p[pi];
  const int blk = blockIdx.x - G.blk0[pi], nblk = G.blk0[pi + 1] - G.blk0[pi];
  const int r0 = blk * P.rpb, r1 = min(P.rows, r0 + P.rpb);
  const Lanes L = lanes_of(P.c);
  float s1[8], s2[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) s1[e] = s2[e] = 0.f;
  const bool act = P.act != PK_CNN_ACT_NONE, store = act || P.g != P.dy;
  auto fold = [&](float (&a)[8], int r) {
    if (store) *reinterpret_cast<uint4*>(bptr(P.g, r, P.ld, L.ch)) = pack8(a);
#pragma unroll
    for (int e = 0; e < 8; ++e) s1[e] += a[e];
  };
  if (act) {
    const uint8_t* const base[2] = {static_cast<const uint8_t*>(P.dy) + 2 * L.ch,
                                    static_cast<const uint8_t*>(P.fout) + 2 * L.ch};
    const size_t pitch[2] = {(size_t)P.ld * 2, (size_t)P.ld * 2};
    row_loop<2>(L, r0, r1, base, pitch, [&](const uint4 (&v)[2], int r) {
      float a[8], fo[8];
      unpack8(v[0], a);
      unpack8(v[1], fo);
#pragma unroll
      for (int e = 0; e < 8; ++e) a[e] *= act_bwd(fo[e], P.act);
      fold(a, r);
    });
  } else {
    const uint8_t* const base[1] = {static_cast<const uint8_t*>(P.dy) + 2 * L.ch};
    const size_t pitch[1] = {(size_t)P.ld * 2};
    row_loop<1>(L, r0, r1, base, pitch, [&](const uint4 (&v)[1], int r) {
      float a[8];
      unpack8(v[0], a);
      fold(a, r);
    });
  }
  block_colsum2(L, P.c, s1, s2, P.ws + (size_t)blk * 2 * P.c);
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
  pdl_gate();
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_reduce& P = G.p[pi];
  const long long i4 = (long long)(blockIdx.x - G.blk0[pi]) * kBlock + threadIdx.x;
  if (i4 * 4 >= P.len) return;
  float4 s = __ldcg(reinterpret_cast<const float4*>(P.src) + i4);
  for (int j0 = 1; j0 < P.splits; j0 += 8) {  // eight partials' loads in flight, summed in order
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (j0 + u < P.splits)
        v[u] = __ldcg(reinterpret_cast<const float4*>(P.src + (long long)(j0 + u) * P.len) + i4);
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (j0 + u < P.splits) {
        s.x += v[u].x; s.y += v[u].y; s.z += v[u].z; s.w += v[u].w;
      }
  }
  reinterpret_cast<float4*>(P.dst)[i4] = s;
  if (!isfinite(s.x) || !isfinite(s.y) || !isfinite(s.z) || !isfinite(s.w)) *P.flag = 1;
}

// ====================== fused multi-member optimizer (K7) ==========================
// reference engine.py:295-326 (+ coupled weight decay g += wd·w, the torch.optim
// rule, as the north_star's per-member extension).  A flagged member (non-finite
// gradient anywhere) is left untouched, engine.py:297-299.
constexpr int kOptChunk = 4096;  // elements per block
__device__ __forceinline__ uint32_t tc_pack_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);  // .x = lo (low half), .y = hi
  return *reinterpret_cast<uint32_t*>(&h);
}
__global__ void __launch_bounds__(kBlock, 4) k_opt(const pk_cnn_opt_seg* segs, const int* blk0,
                                                int nseg) {
  pdl_gate();
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
  // full, 16-byte-aligned chunks: every thread's four float4 groups of each stream
  // are loaded before any update is stored (the scalar loop below serialises a
  // round trip per element, since its stores may alias the next loads); the same
  // per-element arithmetic, so the results are identical
  const bool al = ((reinterpret_cast<uintptr_t>(S.w) | reinterpret_cast<uintptr_t>(S.g) |
                    reinterpret_cast<uintptr_t>(S.s1) | reinterpret_cast<uintptr_t>(S.s2) |
                    reinterpret_cast<uintptr_t>(S.w16)) & 15) == 0;
  if (al && base + kOptChunk <= S.len) {
    constexpr int NV = 2;  // float4 groups per thread in flight (two passes per chunk)
    const bool one = S.kind != PK_OPT_SGD, two = S.kind == PK_OPT_ADAM;
#pragma unroll 1
    for (int pass = 0; pass < kOptChunk / (4 * kBlock * NV); ++pass) {
    float4 w[NV], g[NV], a[NV], b[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const long long i = base + 4LL * (threadIdx.x + (pass * NV + j) * kBlock);
      w[j] = *reinterpret_cast<const float4*>(S.w + i);
      g[j] = *reinterpret_cast<const float4*>(S.g + i);
      if (one) a[j] = *reinterpret_cast<const float4*>(S.s1 + i);
      if (two) b[j] = *reinterpret_cast<const float4*>(S.s2 + i);
    }
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      float* wp = &w[j].x;
      float* gp = &g[j].x;
      float* ap = &a[j].x;
      float* bp = &b[j].x;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float wv = wp[e], gv = gp[e];
        if (wd != 0.f) gv = fmaf(wd, wv, gv);
        switch (S.kind) {
          case PK_OPT_SGD:
            wv -= lr * gv;
            break;
          case PK_OPT_MOMENTUM: {
            const float v = 0.9f * ap[e] + gv;
            ap[e] = v;
            wv -= lr * v;
            break;
          }
          case PK_OPT_ADAGRAD: {
            const float acc = ap[e] + gv * gv;
            ap[e] = acc;
            wv -= lr * gv / (sqrtf(acc) + 1e-10f);
            break;
          }
          default: {  // adam
            const float m = 0.9f * ap[e] + 0.1f * gv;
            const float v = 0.999f * bp[e] + 0.001f * (gv * gv);
            ap[e] = m;
            bp[e] = v;
            wv -= lr * (m / c1) / (sqrtf(v / c2) + 1e-8f);
          }
        }
        wp[e] = wv;
      }
      const long long i = base + 4LL * (threadIdx.x + (pass * NV + j) * kBlock);
      *reinterpret_cast<float4*>(S.w + i) = w[j];
      if (one) *reinterpret_cast<float4*>(S.s1 + i) = a[j];
      if (two) *reinterpret_cast<float4*>(S.s2 + i) = b[j];
      if (S.w16) {
        uint2 h;
        h.x = tc_pack_bf16(w[j].x, w[j].y);
        h.y = tc_pack_bf16(w[j].z, w[j].w);
        *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(S.w16) + i) = h;
      }
    }
    }
    return;
  }
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
// 64 x 64 (co x ci) tiles of one tap; 16-byte loads and stores (k, c are
// multiples of 8, so a vector is either inside the matrix or outside it)
constexpr int kTposeTile = 64;
__global__ void __launch_bounds__(kBlock) k_publish_t(const __grid_constant__ Pack<pk_cnn_tpose> G) {
  pdl_gate();
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_tpose& P = G.p[pi];
  const int tk = (P.k + kTposeTile - 1) / kTposeTile, tc = (P.c + kTposeTile - 1) / kTposeTile;
  int b = blockIdx.x - G.blk0[pi];
  const int tap = b / (tk * tc);
  b -= tap * tk * tc;
  const int kt = b / tc, ct = b - kt * tc;
  __shared__ __align__(16) uint16_t tile[kTposeTile][kTposeTile + 8];
  const uint16_t* src = static_cast<const uint16_t*>(P.src);
  uint16_t* dst = static_cast<uint16_t*>(P.dst);
  const int t = threadIdx.x, j = t & 7, r = t >> 3;  // 32 rows x 8 vectors per pass
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int i = r + 32 * h, co = kt * kTposeTile + i, ci = ct * kTposeTile + 8 * j;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (co < P.k && ci < P.c)
      v = __ldg(reinterpret_cast<const uint4*>(src + (long long)co * P.kpad + tap * P.c + ci));
    *reinterpret_cast<uint4*>(&tile[i][8 * j]) = v;
  }
  __syncthreads();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int o = r + 32 * h, ci = ct * kTposeTile + o, co = kt * kTposeTile + 8 * j;
    if (ci >= P.c || co >= P.k) continue;
    uint16_t e[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) e[q] = tile[8 * j + q][o];
    uint4 v;
    v.x = e[0] | ((uint32_t)e[1] << 16);
    v.y = e[2] | ((uint32_t)e[3] << 16);
    v.z = e[4] | ((uint32_t)e[5] << 16);
    v.w = e[6] | ((uint32_t)e[7] << 16);
    *reinterpret_cast<uint4*>(dst + (long long)ci * P.kpadt + tap * P.k + co) = v;
  }
}

// Commit, reference packing.py:250-257 + engine.py:297-299: members are
// updated in pack order and the first non-finite gradient aborts the loop, so a
// member commits only if no member at or before it (in the problem order) is
// flagged.  mode 0 (before the optimizer, one thread): verdict = prefix-OR of
// the flags; mode 1 (after it): step += !verdict, verdict |= flag << 1, flag = 0.
__global__ void k_commit(const pk_cnn_commit* probs, int nprob, int mode) {
  pdl_gate();
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
// Dense im2col (pk_cnn_im2col, c <= 8): a block owns one run of up to kIm2colPix
// output pixels of one output row.  The input window rows that run touches
// (R rows x ((kIm2colPix - 1)·stride + S) columns, one 16-byte channel vector
// each) are staged in shared memory once — every input vector is read from L2
// once per block instead of once per tap — then each thread (tap t % 64, pixel
// lane t / 64) copies its tap's c values into the block's output rows, which
// leave as coalesced 16-byte vectors (zero columns past r·s·c).
constexpr int kIm2colPix = 64, kIm2colStage = 1024;  // staged input vectors <= 16 KB
__host__ __device__ __forceinline__ int im2col_stage_cols(int s, int stride) {
  return (kIm2colPix - 1) * stride + s;
}
__global__ void __launch_bounds__(kBlock) k_im2col(const __grid_constant__ Pack<pk_cnn_im2col> G) {
  pdl_gate();
  const int pi = pack_prob(G, blockIdx.x);
  const pk_cnn_im2col& P = G.p[pi];
  __shared__ __align__(16) __nv_bfloat16 rows[kIm2colPix * 256];  // ldo <= 256
  __shared__ __align__(16) uint4 stage[kIm2colStage];
  const int taps = P.r * P.s, kr = taps * P.c;
  const int segs = (P.q + kIm2colPix - 1) / kIm2colPix;
  int b = blockIdx.x - G.blk0[pi];
  const int seg = b % segs;
  b /= segs;
  const int oy = b % P.p, n = b / P.p;
  const int ox0 = seg * kIm2colPix, np = min(kIm2colPix, P.q - ox0);
  const int iy0 = oy * P.stride - P.pad, ix0 = ox0 * P.stride - P.pad;
  const int W = im2col_stage_cols(P.s, P.stride);
  const int t = threadIdx.x;
  const uint8_t* src = static_cast<const uint8_t*>(P.src);
  const size_t pitch = (size_t)P.cp * 2;
  for (int i = t; i < P.r * W; i += kBlock) {  // the window rows, zero outside the plane
    const int rr = i / W, cx = i - rr * W, iy = iy0 + rr, ix = ix0 + cx;
    stage[i] = (unsigned)iy < (unsigned)P.h && (unsigned)ix < (unsigned)P.w
                   ? ldg16(src + ((size_t)(n * P.h + iy) * P.w + ix) * pitch)
                   : make_uint4(0, 0, 0, 0);
  }
  for (int i = t; i < np * (P.ldo - kr); i += kBlock) {
    const int pl = i / (P.ldo - kr);
    rows[pl * P.ldo + kr + (i - pl * (P.ldo - kr))] = __float2bfloat16(0.f);
  }
  __syncthreads();
  for (int tap = t & 63; tap < taps; tap += 64) {
    const int rr = tap / P.s, ss = tap - rr * P.s;
    for (int pl = t >> 6; pl < np; pl += 4) {
      const uint4 v = stage[rr * W + pl * P.stride + ss];
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
      uint16_t* d = reinterpret_cast<uint16_t*>(rows) + pl * P.ldo + tap * P.c;
#pragma unroll
      for (int ch = 0; ch < 8; ++ch)
        if (ch < P.c) d[ch] = (uint16_t)(w[ch >> 1] >> (16 * (ch & 1)));
    }
  }
  __syncthreads();
  const int vpr = P.ldo >> 3;  // 16-byte vectors per row
  const long long m0 = ((long long)n * P.p + oy) * P.q + ox0;
  uint4* dst = reinterpret_cast<uint4*>(static_cast<uint8_t*>(P.dst) + m0 * P.ldo * 2);
  const uint4* sv = reinterpret_cast<const uint4*>(rows);
  for (int i = t; i < np * vpr; i += kBlock) dst[i] = sv[i];
}

__global__ void __launch_bounds__(kBlock) k_gather(const __grid_constant__ Pack<pk_cnn_gather> G) {
  pdl_gate();
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
