// pk_kernels.cuh — sm_100a kernels of the packed MLP train step.
//
// One packed step = FWD(l) for l = 0..Lmax-1  →  HEAD  →  BWD(l) for
// l = Lmax-1..0  →  FINALIZE, each a single grouped launch over all members
// (reference: packing.py:185-264 → engine.forward :180-238, backward
// :241-292, apply_update :295-326).
//
//  * FWD tiles compute Z = A·W + b and A' = act(Z) for a [32 x 16] block of
//    one member's layer; layer 0 reads its rows straight from the device
//    dataset through the epoch order (shared-input gather, data.py:131-136
//    fused; members of one input group read the same rows, which stay L2
//    resident, so the batch is fetched from HBM once per group).
//  * BWD tiles are of two kinds in the same launch: DGRAD tiles produce the
//    next gradient dZ_{l-1} = (dZ_l·W_lᵀ) ⊙ act'(Z_{l-1}); WGRAD tiles form
//    dW_l = A_{l-1}ᵀ·dZ_l (and db_l) in shared memory and apply the member's
//    optimizer in the epilogue, so the gradient never touches HBM.  The
//    update writes the member's *other* parameter/slot buffer (ping-pong),
//    which (a) removes the WAR hazard with DGRAD reading the old W in the
//    same launch and (b) lets FINALIZE commit or drop a member's update
//    atomically after the finite checks (engine.py:297-299 semantics).
//  * Every output element is reduced in an order fixed by the layer's shape
//    only (chunk = SK·BK, slice order 0..SK-1), never by K or by which other
//    members share the launch, so a member's packed trajectory is
//    bit-identical to its standalone one (tests/test_pack.py:57-82).
#pragma once

#include <cstdint>
#include <climits>
#include <cuda_runtime.h>

#include "packtrain_b200.h"

namespace pk {

constexpr int NT = 256;  // threads per CTA for every tile kernel

enum TileKind : int16_t { TK_FWD = 0, TK_DGRAD = 1, TK_WGRAD = 2 };

// device-resident per-member control block
struct MemberCtl {
  int32_t parity;      // which params/slots buffer is committed
  int32_t bad_node;    // min non-finite forward node index, INT_MAX = none
  int32_t bad_grad;    // min non-finite grad position, INT_MAX = none
  int32_t fault_grad;  // testing hook: poison this grad position (-1 none)
  int64_t step_counter;
  double lr;
  double loss;         // last step loss
  double eval_acc;     // eval: running sum of per-row losses
};

template <typename T>
struct MemberDev {
  int32_t n_layers, act, opt, max_rows;
  int32_t dims[PK_MAX_LAYERS + 1];
  int32_t n_slots, pad0;
  double wd;
  int64_t n_params;
  int64_t w_off[PK_MAX_LAYERS];
  int64_t b_off[PK_MAX_LAYERS];
  T* params[2];
  T* slots[2];  // [n_slots][n_params] per buffer
  T* Z[PK_MAX_LAYERS];   // pre-activation  [max_rows][dims[l+1]]
  T* A[PK_MAX_LAYERS];   // post-activation [max_rows][dims[l+1]] (hidden)
  T* dZ[PK_MAX_LAYERS];  // dLoss/dZ_l      [max_rows][dims[l+1]]
  MemberCtl* ctl;
};

template <typename T>
struct FeedDev {
  const T* feat;          // dataset features [n][ld]
  const int32_t* labels;  // dataset labels [n]
  const int32_t* rows;    // order + pos, or nullptr (identity from row0)
  int64_t row0;
  int32_t ld;
  int32_t take;           // 0 = inactive
};

struct Tile {
  int32_t member;
  int16_t layer;
  int16_t kind;
  int32_t m0, n0;
};

struct StepHdr {
  int32_t K;
  int32_t slot;   // result ring slot (host-mapped)
  int32_t mode;   // 0 train, 1 eval chunk (no backward, accumulate losses)
  int32_t pad;
};

// -------------------------------------------------------------- math ----

__device__ __forceinline__ bool finite(float v) { return isfinite(v); }
__device__ __forceinline__ bool finite(double v) { return isfinite(v); }
__device__ __forceinline__ float ex(float v) { return expf(v); }
__device__ __forceinline__ double ex(double v) { return exp(v); }
__device__ __forceinline__ float lg(float v) { return logf(v); }
__device__ __forceinline__ double lg(double v) { return log(v); }
__device__ __forceinline__ float th(float v) { return tanhf(v); }
__device__ __forceinline__ double th(double v) { return tanh(v); }
__device__ __forceinline__ float sq(float v) { return sqrtf(v); }
__device__ __forceinline__ double sq(double v) { return sqrt(v); }

// engine.py:202-210
template <typename T>
__device__ __forceinline__ T act_fwd(int act, T z) {
  switch (act) {
    case PK_ACT_SIGMOID: return T(1) / (T(1) + ex(-z));
    case PK_ACT_TANH: return th(z);
    case PK_ACT_RELU: return z > T(0) ? z : T(0);
    default: return z >= T(0) ? z : T(0.01) * z;  // leaky_relu, slope :14
  }
}

// engine.py:274-290 — relu keys on z > 0, leaky on z >= 0; sigmoid/tanh
// use the stored output a.
template <typename T>
__device__ __forceinline__ T act_bwd(int act, T z, T a, T d) {
  switch (act) {
    case PK_ACT_SIGMOID: return d * a * (T(1) - a);
    case PK_ACT_TANH: return d * (T(1) - a * a);
    case PK_ACT_RELU: return z > T(0) ? d : d * T(0);
    default: return d * (z >= T(0) ? T(1) : T(0.01));
  }
}

// engine.py:302-324 for one element; returns the new weight.  c = current
// buffer, n = next buffer.  bc1/bc2 are Adam's bias corrections for t.
template <typename T>
__device__ __forceinline__ void opt_apply(int opt, T lr, T wd, T bc1, T bc2,
                                          const T* __restrict__ wc, T* __restrict__ wn,
                                          const T* __restrict__ s0c, T* __restrict__ s0n,
                                          const T* __restrict__ s1c, T* __restrict__ s1n,
                                          int64_t i, T g) {
  T w = wc[i];
  if (wd != T(0)) g = g + wd * w;
  switch (opt) {
    case PK_OPT_SGD:
      wn[i] = w - lr * g;
      break;
    case PK_OPT_MOMENTUM: {
      T v = s0c[i] * T(0.9) + g;
      s0n[i] = v;
      wn[i] = w - lr * v;
      break;
    }
    case PK_OPT_ADAGRAD: {
      T a = s0c[i] + g * g;
      s0n[i] = a;
      wn[i] = w - lr * g / (sq(a) + T(1e-10));
      break;
    }
    default: {  // adam
      T m = s0c[i] * T(0.9) + (T(1) - T(0.9)) * g;
      T v = s1c[i] * T(0.999) + (T(1) - T(0.999)) * g * g;
      s0n[i] = m;
      s1n[i] = v;
      wn[i] = w - lr * (m / bc1) / (sq(v / bc2) + T(1e-8));
      break;
    }
  }
}

// ------------------------------------------------------- tile GEMM core --
//
// C[m][n] = Σ_k A(m,k)·B(k,n) over a BM x BN tile; the reduction runs in
// chunks of SK·BK, slice s of the CTA taking sub-chunk s.  Partial tiles are
// left in shared memory `red[SK][BM][BN]`; the caller's epilogue sums them in
// slice order.  A(m,k) / B(k,n) are fetched by functors; AKF / BKF say
// whether k is the contiguous (fast) index in global memory.

template <typename T, int BM, int BN, int BK, int SK, int TM, int TN>
struct TileGemm {
  static constexpr int TPS = NT / SK;
  static constexpr int RS = BM / TM;  // row stride inside a thread's micro-tile
  static constexpr int CS = BN / TN;
  static_assert(RS * CS == TPS, "micro-tile does not cover the tile");
  static constexpr int KC = SK * BK;  // reduction chunk
  static constexpr int LDA = BM + 1, LDB = BN + 1;
  static constexpr int STAGE = KC * LDA + KC * LDB;
  static constexpr int RED = SK * BM * BN;
  static constexpr int SMEM = (STAGE > RED ? STAGE : RED);

  template <bool KFAST, int MM, int LD, class F>
  __device__ __forceinline__ static bool stage(T* S, F get, int k0, int m0, int kmax,
                                               int mmax) {
    bool bad = false;
#pragma unroll 4
    for (int e = threadIdx.x; e < KC * MM; e += NT) {
      int kk, mm;
      if (KFAST) { kk = e % KC; mm = e / KC; }
      else { mm = e % MM; kk = e / MM; }
      const int k = k0 + kk, m = m0 + mm;
      T v = T(0);
      if (k < kmax && m < mmax) {
        v = get(m, k);
        bad |= !finite(v);
      }
      S[kk * LD + mm] = v;
    }
    return bad;
  }

  // returns (block-wide) whether any staged A element was non-finite
  template <bool AKF, bool BKF, class FA, class FB>
  __device__ __forceinline__ static bool run(T* smem, FA getA, FB getB, int m0, int n0, int M,
                                             int N, int Kred) {
    T* As = smem;
    T* Bs = smem + KC * LDA;
    const int slice = threadIdx.x / TPS, lt = threadIdx.x % TPS;
    const int tc = lt % CS, tr = lt / CS;
    T acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j] = T(0);
    bool badA = false;
    for (int k0 = 0; k0 < Kred; k0 += KC) {
      badA |= stage<AKF, BM, LDA>(As, getA, k0, m0, Kred, M);
      stage<BKF, BN, LDB>(Bs, getB, k0, n0, Kred, N);
      __syncthreads();
      const T* a_s = As + (slice * BK) * LDA + tr;
      const T* b_s = Bs + (slice * BK) * LDB + tc;
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        T a[TM], b[TN];
#pragma unroll
        for (int i = 0; i < TM; ++i) a[i] = a_s[kk * LDA + i * RS];
#pragma unroll
        for (int j = 0; j < TN; ++j) b[j] = b_s[kk * LDB + j * CS];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
      }
      __syncthreads();
    }
    T* red = smem + slice * (BM * BN);
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) red[(tr + i * RS) * BN + tc + j * CS] = acc[i][j];
    return __syncthreads_or(badA);
  }

  // reduced value of tile element (mm, nn), fixed slice order
  __device__ __forceinline__ static T value(const T* smem, int mm, int nn) {
    T v = smem[mm * BN + nn];
#pragma unroll
    for (int s = 1; s < SK; ++s) v += smem[s * BM * BN + mm * BN + nn];
    return v;
  }
};

// tile shapes (fixed per kernel kind, never per pack → K-invariant)
template <typename T> using FwdGemm = TileGemm<T, 32, 16, 8, 8, 4, 4>;
template <typename T> using DgradGemm = TileGemm<T, 32, 16, 8, 8, 4, 4>;
template <typename T> using WgradGemm = TileGemm<T, 32, 32, 8, 4, 4, 4>;
constexpr int FWD_BM = 32, FWD_BN = 16;
constexpr int DG_BM = 32, DG_BN = 16;
constexpr int WG_BM = 32, WG_BN = 32;

__device__ __forceinline__ void flag_min(int32_t* p, int v) { atomicMin(p, v); }

// ------------------------------------------------------------- kernels --

template <typename T>
struct SmemBuf {
  static constexpr int N =
      (FwdGemm<T>::SMEM > WgradGemm<T>::SMEM ? FwdGemm<T>::SMEM : WgradGemm<T>::SMEM);
};

// Forward of layer `t.layer` for one [32 x 16] output tile.
template <typename T>
__device__ __forceinline__ void fwd_tile(T* smem, const MemberDev<T>& M, const FeedDev<T>& f,
                                         const Tile& t) {
  using G = FwdGemm<T>;
  const int l = t.layer, in = M.dims[l], out = M.dims[l + 1];
  const int R = f.take;
  const int par = M.ctl->parity;
  const T* W = M.params[par] + M.w_off[l];
  const T* bias = M.params[par] + M.b_off[l];
  auto getB = [&](int n, int k) { return W[(int64_t)k * out + n]; };
  bool badX;
  if (l == 0) {
    const T* X = f.feat;
    const int32_t* rows = f.rows;
    const int64_t row0 = f.row0, ld = f.ld;
    auto getA = [&](int m, int k) {
      const int64_t r = rows ? (int64_t)rows[m] : row0 + m;
      return X[r * ld + k];
    };
    badX = G::template run<true, false>(smem, getA, getB, t.m0, t.n0, R, out, in);
  } else {
    const T* Ain = M.A[l - 1];
    auto getA = [&](int m, int k) { return Ain[(int64_t)m * in + k]; };
    badX = G::template run<true, false>(smem, getA, getB, t.m0, t.n0, R, out, in);
    badX = false;  // hidden inputs were checked where they were produced
  }
  const bool last = (l == M.n_layers - 1);
  T* Z = M.Z[l];
  T* A = M.A[l];
  int bad = INT_MAX;
  for (int e = threadIdx.x; e < FWD_BM * FWD_BN; e += NT) {
    const int mm = e / FWD_BN, nn = e % FWD_BN;
    const int m = t.m0 + mm, n = t.n0 + nn;
    if (m >= R || n >= out) continue;
    const T z = G::value(smem, mm, nn) + bias[n];
    Z[(int64_t)m * out + n] = z;
    if (!finite(z)) bad = min(bad, 1 + 2 * l);
    if (!last) {
      const T a = act_fwd(M.act, z);
      A[(int64_t)m * out + n] = a;
      if (!finite(a)) bad = min(bad, 2 + 2 * l);
    }
  }
  if (badX && threadIdx.x == 0) flag_min(&M.ctl->bad_node, 0);
  if (bad != INT_MAX) flag_min(&M.ctl->bad_node, bad);
}

template <typename T>
__global__ void __launch_bounds__(NT) k_fwd(const MemberDev<T>* __restrict__ mems,
                                            const FeedDev<T>* __restrict__ feeds,
                                            const Tile* __restrict__ tiles) {
  __shared__ __align__(16) T smem[SmemBuf<T>::N];
  const Tile t = tiles[blockIdx.x];
  const FeedDev<T> f = feeds[t.member];
  if (f.take == 0 || t.m0 >= f.take) return;
  fwd_tile<T>(smem, mems[t.member], f, t);
}

// DGRAD: dZ_{l-1}[r][i] = act'(Z,A)[r][i] · Σ_j dZ_l[r][j] W_l[i][j]
template <typename T>
__device__ __forceinline__ void dgrad_tile(T* smem, const MemberDev<T>& M, const FeedDev<T>& f,
                                           const Tile& t) {
  using G = DgradGemm<T>;
  const int l = t.layer, in = M.dims[l], out = M.dims[l + 1];
  const int R = f.take;
  const int par = M.ctl->parity;
  const T* W = M.params[par] + M.w_off[l];
  const T* dZ = M.dZ[l];
  auto getA = [&](int m, int k) { return dZ[(int64_t)m * out + k]; };
  auto getB = [&](int n, int k) { return W[(int64_t)n * out + k]; };
  G::template run<true, true>(smem, getA, getB, t.m0, t.n0, R, in, out);
  const T* Zp = M.Z[l - 1];
  const T* Ap = M.A[l - 1];
  T* dZp = M.dZ[l - 1];
  for (int e = threadIdx.x; e < DG_BM * DG_BN; e += NT) {
    const int mm = e / DG_BN, nn = e % DG_BN;
    const int m = t.m0 + mm, n = t.n0 + nn;
    if (m >= R || n >= in) continue;
    const int64_t o = (int64_t)m * in + n;
    dZp[o] = act_bwd(M.act, Zp[o], Ap[o], G::value(smem, mm, nn));
  }
}

// WGRAD + optimizer: W_l' = opt(W_l, A_{l-1}ᵀ·dZ_l); tiles with m0 == 0 also
// reduce and update the bias.  Grad finiteness is flagged per tensor.
template <typename T>
__device__ __forceinline__ void wgrad_tile(T* smem, const MemberDev<T>& M, const FeedDev<T>& f,
                                           const Tile& t) {
  using G = WgradGemm<T>;
  const int l = t.layer, in = M.dims[l], out = M.dims[l + 1];
  const int R = f.take;
  const int par = M.ctl->parity;
  const T* dZ = M.dZ[l];
  auto getB = [&](int n, int k) { return dZ[(int64_t)k * out + n]; };
  if (l == 0) {
    const T* X = f.feat;
    const int32_t* rows = f.rows;
    const int64_t row0 = f.row0, ld = f.ld;
    auto getA = [&](int m, int k) {
      const int64_t r = rows ? (int64_t)rows[k] : row0 + k;
      return X[r * ld + m];
    };
    G::template run<false, false>(smem, getA, getB, t.m0, t.n0, in, out, R);
  } else {
    const T* Ain = M.A[l - 1];
    auto getA = [&](int m, int k) { return Ain[(int64_t)k * in + m]; };
    G::template run<false, false>(smem, getA, getB, t.m0, t.n0, in, out, R);
  }
  const MemberCtl* ctl = M.ctl;
  const T lr = T(ctl->lr), wd = T(M.wd);
  T bc1 = T(1), bc2 = T(1);
  if (M.opt == PK_OPT_ADAM) {
    const double tt = double(ctl->step_counter + 1);
    bc1 = T(1.0 - pow(0.9, tt));
    bc2 = T(1.0 - pow(0.999, tt));
  }
  const int64_t P = M.n_params;
  const T* wc = M.params[par];
  T* wn = M.params[par ^ 1];
  const T* sc = M.slots[par];
  T* sn = M.slots[par ^ 1];
  const T* s0c = sc; T* s0n = sn;
  const T* s1c = sc ? sc + P : nullptr; T* s1n = sn ? sn + P : nullptr;
  const int gpos = 2 * (M.n_layers - 1 - l);
  bool badW = false, badB = false;
  for (int e = threadIdx.x; e < WG_BM * WG_BN; e += NT) {
    const int mm = e / WG_BN, nn = e % WG_BN;
    const int m = t.m0 + mm, n = t.n0 + nn;
    if (m >= in || n >= out) continue;
    T g = G::value(smem, mm, nn);
    if (ctl->fault_grad == gpos) g = T(NAN);
    badW |= !finite(g);
    opt_apply(M.opt, lr, wd, bc1, bc2, wc, wn, s0c, s0n, s1c, s1n,
              M.w_off[l] + (int64_t)m * out + n, g);
  }
  if (t.m0 == 0 && threadIdx.x < WG_BN) {
    const int n = t.n0 + threadIdx.x;
    if (n < out) {
      T g = T(0);
      for (int r = 0; r < R; ++r) g += dZ[(int64_t)r * out + n];
      if (ctl->fault_grad == gpos + 1) g = T(NAN);
      badB = !finite(g);
      opt_apply(M.opt, lr, wd, bc1, bc2, wc, wn, s0c, s0n, s1c, s1n, M.b_off[l] + n, g);
    }
  }
  if (badW) flag_min(&M.ctl->bad_grad, gpos);
  if (badB) flag_min(&M.ctl->bad_grad, gpos + 1);
}

template <typename T>
__global__ void __launch_bounds__(NT) k_bwd(const MemberDev<T>* __restrict__ mems,
                                            const FeedDev<T>* __restrict__ feeds,
                                            const Tile* __restrict__ tiles) {
  __shared__ __align__(16) T smem[SmemBuf<T>::N];
  const Tile t = tiles[blockIdx.x];
  const FeedDev<T> f = feeds[t.member];
  if (f.take == 0) return;
  if (t.kind == TK_DGRAD) {
    if (t.m0 >= f.take) return;
    dgrad_tile<T>(smem, mems[t.member], f, t);
  } else {
    wgrad_tile<T>(smem, mems[t.member], f, t);
  }
}

// ---------------------------------------------------------------- head --
// Softmax cross-entropy over the member's valid rows (engine.py:211-230,
// :252-264): one CTA per member, one warp per row.  Loss = −mean(logp[y]),
// summed in a fixed order (thread-strided, then a fixed tree) in float64.
template <typename T>
__global__ void __launch_bounds__(NT) k_head(const MemberDev<T>* __restrict__ mems,
                                             const FeedDev<T>* __restrict__ feeds,
                                             const StepHdr* __restrict__ hdr) {
  __shared__ double part[NT];
  const int k = blockIdx.x;
  const FeedDev<T> f = feeds[k];
  const int R = f.take;
  if (R == 0) return;
  const MemberDev<T>& M = mems[k];
  const int L = M.n_layers - 1, C = M.dims[L + 1];
  const T* Zl = M.Z[L];
  T* dZ = M.dZ[L];
  const bool train = (hdr->mode == 0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // per-row loss terms are written to part-of-thread slots in a fixed map:
  // row r is owned by thread (r % NT)'s running sum (rows visited in order)
  double mysum = 0.0;
  for (int r0 = 0; r0 < R; r0 += NT / 32 * 32) {
    // each warp handles 32 consecutive rows of this batch-chunk, one at a time
    for (int rr = 0; rr < 32; ++rr) {
      const int r = r0 + warp * 32 + rr;
      if (r >= R) break;
      const T* z = Zl + (int64_t)r * C;
      T mx = -INFINITY;
      for (int c = lane; c < C; c += 32) mx = max(mx, z[c]);
#pragma unroll
      for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      T s = T(0);
      for (int c = lane; c < C; c += 32) s += ex(z[c] - mx);
#pragma unroll
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      const int64_t src = f.rows ? (int64_t)f.rows[r] : f.row0 + r;
      const int y = f.labels[src];
      if (train) {
        const T inv = T(1) / s;
        const T nv = T(R);
        for (int c = lane; c < C; c += 32) {
          T p = ex(z[c] - mx) * inv;
          if (c == y) p -= T(1);
          dZ[(int64_t)r * C + c] = p / nv;
        }
      }
      if (lane == (r & 31)) {
        const T logp = (z[y] - mx) - lg(s);
        mysum += -(double)logp;
      }
    }
  }
  part[threadIdx.x] = mysum;
  __syncthreads();
  for (int w = NT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    MemberCtl* ctl = M.ctl;
    if (train) {
      const double loss = part[0] / double(R);
      ctl->loss = loss;
      if (!isfinite(loss)) atomicMin(&ctl->bad_node, 2 * M.n_layers);
    } else {
      ctl->eval_acc += part[0];
    }
  }
}

// ------------------------------------------------------------ finalize --
// Commit rules of packing.py:246-253: a forward non-finite value aborts the
// whole step; otherwise members commit in pack order until the first member
// with a non-finite gradient.  Writes {status, losses} to the host ring.
template <typename T>
__global__ void k_finalize(const MemberDev<T>* __restrict__ mems,
                           const FeedDev<T>* __restrict__ feeds,
                           const StepHdr* __restrict__ hdr, char* __restrict__ ring,
                           int32_t ring_stride) {
  if (threadIdx.x != 0) return;
  const int K = hdr->K;
  int32_t* st = reinterpret_cast<int32_t*>(ring + (int64_t)hdr->slot * ring_stride);
  double* losses = reinterpret_cast<double*>(st + 4);
  int code = PK_OK, who = -1, idx = -1, committed = 0;
  for (int k = 0; k < K; ++k) {
    if (!feeds[k].take) continue;
    const int b = mems[k].ctl->bad_node;
    if (b != INT_MAX) { code = PK_ERR_NONFINITE_VALUE; who = k; idx = b; break; }
  }
  for (int k = 0; k < K; ++k) {
    MemberCtl* c = mems[k].ctl;
    const bool act = feeds[k].take != 0;
    losses[k] = act ? c->loss : 0.0;
    if (act && code == PK_OK) {
      if (c->bad_grad != INT_MAX) {
        code = PK_ERR_NONFINITE_GRAD; who = k; idx = c->bad_grad;
      } else {
        c->parity ^= 1;
        c->step_counter += 1;
        ++committed;
      }
    }
  }
  for (int k = 0; k < K; ++k) {
    mems[k].ctl->bad_node = INT_MAX;
    mems[k].ctl->bad_grad = INT_MAX;
    if (feeds[k].take) mems[k].ctl->fault_grad = -1;  // one-shot
  }
  st[0] = code; st[1] = who; st[2] = idx; st[3] = committed;
  __threadfence_system();
}

// eval: after the last chunk, losses[k] = eval_acc / rows and reset
template <typename T>
__global__ void k_eval_finish(const MemberDev<T>* __restrict__ mems, int K, const int64_t rows,
                              char* __restrict__ ring, int32_t slot, int32_t ring_stride) {
  if (threadIdx.x != 0) return;
  int32_t* st = reinterpret_cast<int32_t*>(ring + (int64_t)slot * ring_stride);
  double* losses = reinterpret_cast<double*>(st + 4);
  int code = PK_OK, who = -1, idx = -1;
  for (int k = 0; k < K; ++k) {
    MemberCtl* c = mems[k].ctl;
    losses[k] = c->eval_acc / double(rows);
    if (code == PK_OK && c->bad_node != INT_MAX) {
      code = PK_ERR_NONFINITE_VALUE; who = k; idx = c->bad_node;
    }
    c->eval_acc = 0.0;
    c->bad_node = INT_MAX;
    c->bad_grad = INT_MAX;
  }
  st[0] = code; st[1] = who; st[2] = idx; st[3] = 0;
  __threadfence_system();
}

}  // namespace pk
