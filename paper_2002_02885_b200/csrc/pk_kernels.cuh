// pk_kernels.cuh — sm_100a kernels of the packed MLP train step.
//
// A packed step (reference: packing.py:185-264 → engine.forward :180-238,
// backward :241-292, apply_update :295-326) is a short sequence of *phases*;
// every phase is ONE launch of `k_phase` over a list of tiles drawn from all
// K members (grouped launch), chained with programmatic dependent launch so a
// phase's CTAs start (and prefetch their weights) while the previous phase
// drains.  Tile kinds:
//
//   FWD   Z_l = A_{l-1}·W_l + b_l, A_l = act(Z_l) for a [32 x 8] block; for
//         l = 0 the rows are gathered straight from the device dataset
//         through the epoch order (data.py:131-136 fused): members of one
//         input group read the same rows, so the batch crosses HBM once.
//   TAIL  the member's last layer + softmax-xent + the first backward GEMM
//         for a block of 32 rows: logits, loss terms, dZ_L and
//         dZ_{L-1} = (dZ_L·W_Lᵀ) ⊙ act'(Z_{L-1}) in one CTA (W_L resident in
//         shared memory).
//   HEAD  softmax-xent alone (members whose last layer is too big for TAIL).
//   DGRAD dZ_{l-1} = (dZ_l·W_lᵀ) ⊙ act'(Z_{l-1}).
//   WGRAD dW_l = A_{l-1}ᵀ·dZ_l (+ db_l) formed in shared memory and consumed by
//         the member's optimizer in the epilogue — gradients never reach
//         HBM.  The update writes the member's *other* params/slots buffer
//         (ping-pong): no hazard with DGRAD reading the old W in the same
//         phase, and the commit is a parity flip decided after the finite
//         checks (engine.py:297-299).
//
// The last CTA of the last phase runs FINALIZE (loss reduction, commit rules
// of packing.py:250-253, status + losses into a host-mapped ring).
//
// GEMM tiles stream operands through a multi-stage cp.async pipeline.  Every
// output element is reduced in an order fixed by the tile kind and the
// member's own shape — chunk KC, slice order 0..SK-1 — never by K or by the
// other members, so a member's packed trajectory is bit-identical to its
// standalone one (tests/test_pack.py:57-82).
#pragma once

#include <cstdint>
#include <climits>
#include <type_traits>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "packtrain_b200.h"

namespace pk {

constexpr int NT = 256;        // threads per CTA
constexpr int ROWCAP = 1024;   // rows whose gather index is cached in smem
constexpr int PK_MAX_PACK = 1024;  // members per pack (finalize's flag table)

enum TileKind : int16_t { TK_FWD = 0, TK_TAIL = 1, TK_HEAD = 2, TK_DGRAD = 3, TK_WGRAD = 4 };

struct MemberCtl {
  int32_t parity;      // committed params/slots buffer
  int32_t bad_node;    // min non-finite forward node index, INT_MAX = none
  int32_t bad_grad;    // min non-finite grad position, INT_MAX = none
  int32_t fault_grad;  // testing hook: poison this grad position (-1 none)
  int64_t step_counter;
  double lr;
  double loss;         // last step loss
  double eval_acc;     // eval: running sum of per-row losses
  double bc1, bc2;     // Adam bias corrections 1-β^t for t = step_counter + 1
  double bcn1, bcn2;   // tensor path: the same for t = step_counter + 2 (next commit)
};

// 1 - beta^t in float64, t = the update about to be applied (engine.py:322-323)
__host__ __device__ inline void adam_bias_corrections(int64_t step_counter, double* bc1,
                                                      double* bc2) {
  const double t = double(step_counter + 1);
  *bc1 = 1.0 - pow(0.9, t);
  *bc2 = 1.0 - pow(0.999, t);
}

template <typename T>
struct MemberDev {
  int32_t n_layers, act, opt, max_rows;
  int32_t dims[PK_MAX_LAYERS + 1];
  int32_t n_slots, tail;  // tail: last layer handled by a TAIL tile
  int32_t tensor, pad_;   // tensor: pk_m1t.cuh step (loss + next bc from the bwd owner CTA)
  double wd;
  int64_t n_params;
  int64_t s_stride;      // elements between optimizer slot blocks (P rounded to 16 B)
  int64_t w_off[PK_MAX_LAYERS];
  int64_t b_off[PK_MAX_LAYERS];
  T* params[2];
  T* slots[2];  // [n_slots][s_stride] per buffer
  T* Z[PK_MAX_LAYERS];   // pre-activation  [max_rows][dims[l+1]]
  T* A[PK_MAX_LAYERS];   // post-activation [max_rows][dims[l+1]] (hidden)
  T* dZ[PK_MAX_LAYERS];  // dLoss/dZ_l      [max_rows][dims[l+1]]
  double* rowloss;       // per-row −log p[y]  [max_rows]
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

constexpr int kInlineFeeds = 32;  // packs up to this K take inline step descriptors
constexpr int kInlineTiles = 160; // phases up to this many CTAs carry their tiles inline
constexpr int kInlineMems = 4;    // packs up to this K carry member descriptors inline

struct StepHdr {
  int32_t K;
  int32_t slot;   // result ring slot (host-mapped)
  int32_t mode;   // 0 train, 1 eval chunk (forward + loss terms only)
  int32_t pad;
};

template <typename T>
struct PhaseArgs {
  const MemberDev<T>* mems;
  const FeedDev<T>* feeds;
  const StepHdr* hdr;
  const Tile* tiles;
  int32_t* done;       // CTA-completion counter (last phase)
  int32_t* halt;       // set by FINALIZE after a failed train step: later
                       // in-flight train steps skip all work (packed_run)
  char* ring;          // host-mapped results
  int32_t ring_stride;
  int32_t K;
  int32_t is_last;     // run FINALIZE in the last CTA
  int32_t prefetch;    // issue L2 prefetch of params/slots (first phase)
  int32_t first;       // first launch of a step: inside a multi-step graph it waits
                       // for the previous step (PDL) before touching member state
  unsigned long long* trace;  // profiling: kTraceSlots stamps per CTA, or nullptr
  int32_t cs;          // cluster size of this launch (k_m1t_fwd: input splits)
  int32_t stages;      // k_m1t_bwd: input-tile stages in flight
  int32_t gsize;       // k_m1t_bwd: input tiles per group (G)
  // > 0: the step header and the first `nin` feeds travel inline in the kernel
  // parameters (the train graph's kernel nodes are re-parameterised per step:
  // no descriptor copy, feed reads hit the constant bank)
  int32_t nin;
  StepHdr hdr_in;
  FeedDev<T> feeds_in[kInlineFeeds];
  // finalize fast path (K <= kInlineFeeds, every member on the tensor path):
  // the members' control blocks, inline
  int32_t all_tensor;
  MemberCtl* ctl_in[kInlineFeeds];
  // static per phase / pack, inline when small: a CTA's first reads hit the
  // constant bank instead of dependent global loads
  int32_t tin, min_;
  Tile tiles_in[kInlineTiles];
  MemberDev<T> mems_in[kInlineMems];
};

template <typename T>
__device__ __forceinline__ bool halted(const PhaseArgs<T>& P) {
  return P.halt && hdr_of(P).mode == 0 && *reinterpret_cast<volatile int32_t*>(P.halt) != 0;
}

template <typename T>
__device__ __forceinline__ Tile tile_of(const PhaseArgs<T>& P) {
  return P.tin ? P.tiles_in[blockIdx.x] : P.tiles[blockIdx.x];
}
template <typename T>
__device__ __forceinline__ const MemberDev<T>* mem_of(const PhaseArgs<T>& P, int k) {
  return P.min_ ? &P.mems_in[k] : P.mems + k;
}

template <typename T>
__device__ __forceinline__ FeedDev<T> feed_of(const PhaseArgs<T>& P, int k) {
  return P.nin ? P.feeds_in[k] : P.feeds[k];
}
template <typename T>
__device__ __forceinline__ StepHdr hdr_of(const PhaseArgs<T>& P) {
  return P.nin ? P.hdr_in : *P.hdr;
}

// ---- stage tracing (profiling builds of a step, PK_TRACE=1) -------------
// Thread 0 of a CTA stamps %globaltimer at stage boundaries:
//   0 entry, 1 operands/prologue ready, 2 GEMM done, 3 epilogue part 1,
//   4 epilogue part 2, 5 tile done, 6 finalize start, 7 finalize end,
//   8..15 kernel-specific sub-stages (pk_m1t.cuh).
constexpr int kTraceSlots = 16;  // 8..15: kernel-specific sub-stages
__shared__ unsigned long long* pk_trace_slots;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define PK_TRACE(i)                                         \
  do {                                                      \
    if (threadIdx.x == 0) {                                 \
      /* volatile: the load may not be hoisted above the tid test */ \
      unsigned long long* pk_ts_ = *(unsigned long long* volatile*)&pk_trace_slots; \
      if (pk_ts_) pk_ts_[(i)] = gtimer();                   \
    }                                                       \
  } while (0)

// ------------------------------------------------------------ PTX glue --

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;"); }
// kernel entry: a step's first launch waits for the previous step of a
// multi-step graph (its parameters, parity and halt flag) before letting its
// own dependents start; later launches release their dependents at once
#define pdl_begin(P)        \
  do {                      \
    if ((P).first) pdl_wait(); \
    pdl_launch();           \
  } while (0)

template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem, const void* gmem, bool pred) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  const int n = pred ? BYTES : 0;  // src-size 0 → zero fill
  if constexpr (BYTES == 16)  // L2 only: with most of the SM's SRAM carved out as shared
    // memory, L1-allocating copies (.ca) thrash the small L1 and throttle issue
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(s), "l"(gmem),
                 "n"(BYTES), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// one line toward L1 (non-blocking): a step's first kernel touches the halt
// flag, the member's control block and the batch's gather index before any
// of them is used — prefetched together they cost one round trip, not three
__device__ __forceinline__ void l1_prefetch(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
template <typename T>
__device__ __forceinline__ void first_touch(const PhaseArgs<T>& P, const MemberDev<T>* m,
                                            const FeedDev<T>& f) {
  if (threadIdx.x == 0) {
    if (P.halt) asm volatile("prefetch.global.L2 [%0];" ::"l"(P.halt));  // read volatile: L2
    l1_prefetch(m->ctl);
  }
  if (f.rows && (int)threadIdx.x < f.take && (threadIdx.x & 31) == 0) l1_prefetch(f.rows + threadIdx.x);
}

// a small global range toward L2 with one plain prefetch per 128-B line —
// for row segments: small bulk prefetches queue one after another in the
// SM's TMA unit (256 per tile cost the Adam members of k16 ~3 µs per tile)
__device__ __forceinline__ void l2_prefetch_lines(const void* p, uint32_t bytes) {
  const char* a = reinterpret_cast<const char*>(reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)127);
  const char* e = reinterpret_cast<const char*>(p) + bytes;
  for (; a < e; a += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
}

// bulk (TMA-engine) prefetch of a global range into L2
__device__ __forceinline__ void l2_prefetch(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}

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

// engine.py:274-290 — relu keys on z > 0, leaky on z >= 0; sigmoid/tanh use
// the stored output a.
template <typename T>
__device__ __forceinline__ T act_bwd(int act, T z, T a, T d);
// fp32: explicit roundings (no contraction) — bit-identical in every kernel copy
template <>
__device__ __forceinline__ float act_bwd<float>(int act, float z, float a, float d) {
  switch (act) {
    case PK_ACT_SIGMOID: return __fmul_rn(__fmul_rn(d, a), __fsub_rn(1.f, a));
    case PK_ACT_TANH: return __fmul_rn(d, __fsub_rn(1.f, __fmul_rn(a, a)));
    case PK_ACT_RELU: return z > 0.f ? d : __fmul_rn(d, 0.f);
    default: return __fmul_rn(d, z >= 0.f ? 1.f : 0.01f);
  }
}
template <typename T>
__device__ __forceinline__ T act_bwd(int act, T z, T a, T d) {
  switch (act) {
    case PK_ACT_SIGMOID: return d * a * (T(1) - a);
    case PK_ACT_TANH: return d * (T(1) - a * a);
    case PK_ACT_RELU: return z > T(0) ? d : d * T(0);
    default: return d * (z >= T(0) ? T(1) : T(0.01));
  }
}

// engine.py:302-324 for one element, on registers: w, s0, s1 in/out
// (s0 = velocity | accum | m, s1 = v); bc1/bc2 are Adam's bias corrections
template <typename T>
__device__ __forceinline__ void opt_step(int opt, T lr, T wd, T bc1, T bc2, T& w, T& s0, T& s1,
                                         T g) {
  if (wd != T(0)) g = g + wd * w;
  switch (opt) {
    case PK_OPT_SGD:
      w = w - lr * g;
      break;
    case PK_OPT_MOMENTUM:
      s0 = s0 * T(0.9) + g;
      w = w - lr * s0;
      break;
    case PK_OPT_ADAGRAD:
      s0 = s0 + g * g;
      w = w - lr * g / (sq(s0) + T(1e-10));
      break;
    default:  // adam
      s0 = s0 * T(0.9) + (T(1) - T(0.9)) * g;
      s1 = s1 * T(0.999) + (T(1) - T(0.999)) * g * g;
      w = w - lr * (s0 / bc1) / (sq(s1 / bc2) + T(1e-8));
      break;
  }
}

// ------------------------------------------------------- GEMM tile core --
//
// C[m][n] = Σ_k A(m,k)·B(k,n) for one BM x BN tile.  Operands are row-major
// matrices read through `Mat` (row r lives at base + idx(r)·ld, idx from an
// optional gather list).  AK/BK say whether k is the matrix's column
// (contiguous) index: A(m,k) = M[m][k] if AK else M[k][m]; B(k,n) = M[n][k]
// if BK else M[k][n].  Shared-memory stage layouts follow the global ones so
// cp.async copies straight through; STAGES chunks of KC are in flight.
// Slice s of the CTA reduces sub-chunk s; partial tiles end in shared memory
// and value() sums them in slice order.

template <typename T>
struct Mat {
  const T* base;
  const int32_t* rows;  // gather list for the row index, or nullptr
  int64_t row0;         // identity offset when rows == nullptr
  int64_t ld;
};

template <typename T, int BM, int BN, int KC, int TM, int TN, int SK, int STAGES, bool AK, bool BK>
struct Gemm {
  static constexpr int TPS = NT / SK;
  static constexpr int KCH = KC;
  static constexpr int RS = BM / TM;
  static constexpr int CS = BN / TN;
  static_assert(RS * CS == TPS, "micro-tile does not cover the tile");
  static_assert(KC % SK == 0, "chunk not divisible by slices");
  static constexpr int KS = KC / SK;
  static constexpr int A_ELEMS = BM * KC, B_ELEMS = BN * KC;
  static constexpr int VEC = 16 / (int)sizeof(T);  // elements per 16-byte cp.async
  // smem rows padded by one 16-byte vector: keeps vector alignment and
  // spreads the k-major reads of consecutive rows over different banks
  static constexpr int A_LD = AK ? KC + VEC : BM + VEC;
  static constexpr int B_LD = BK ? KC + VEC : BN + VEC;
  static constexpr int A_STAGE = AK ? BM * A_LD : KC * A_LD;
  static constexpr int B_STAGE = BK ? BN * B_LD : KC * B_LD;
  static constexpr int PIPE = STAGES * (A_STAGE + B_STAGE);
  static constexpr int RED = SK * BM * BN;
  static constexpr int SMEM_T = PIPE > RED ? PIPE : RED;  // in elements of T

  // gather offsets for the gathered dimension of A (m if AK, k otherwise)
  __device__ __forceinline__ static int64_t a_row(const Mat<T>& a, const int32_t* srow, int r) {
    if (!a.rows) return (a.row0 + r) * a.ld;
    return (int64_t)(r < ROWCAP ? srow[r] : a.rows[r]) * a.ld;
  }

  // 16-byte path: the contiguous dimension is walked in VEC-element vectors;
  // the caller guarantees alignment and that extents are VEC multiples
  __device__ __forceinline__ static void load_chunk_vec(T* sA, T* sB, const Mat<T>& a,
                                                        const Mat<T>& b, const int32_t* srow,
                                                        int k0, int m0, int n0, int M, int N,
                                                        int Kr, bool va, bool vb, bool do_a = true,
                                                        bool do_b = true) {
    if (va && do_a) {
      for (int e = threadIdx.x; e < A_ELEMS / VEC; e += NT) {
        int kk, mm;
        if (AK) { kk = (e % (KC / VEC)) * VEC; mm = e / (KC / VEC); }
        else { mm = (e % (BM / VEC)) * VEC; kk = e / (BM / VEC); }
        const int k = k0 + kk, m = m0 + mm;
        const bool ok = (k < Kr) && (m < M);
        const T* g = a.base;
        if (ok) g = AK ? a.base + a_row(a, srow, m) + k : a.base + a_row(a, srow, k) + m;
        T* s = AK ? sA + mm * A_LD + kk : sA + kk * A_LD + mm;
        cp_async<16>(s, g, ok);
      }
    }
    if (vb && do_b) {
      for (int e = threadIdx.x; e < B_ELEMS / VEC; e += NT) {
        int kk, nn;
        if (BK) { kk = (e % (KC / VEC)) * VEC; nn = e / (KC / VEC); }
        else { nn = (e % (BN / VEC)) * VEC; kk = e / (BN / VEC); }
        const int k = k0 + kk, n = n0 + nn;
        const bool ok = (k < Kr) && (n < N);
        const T* g = b.base;
        if (ok) g = BK ? b.base + (int64_t)n * b.ld + k : b.base + (int64_t)k * b.ld + n;
        T* s = BK ? sB + nn * B_LD + kk : sB + kk * B_LD + nn;
        cp_async<16>(s, g, ok);
      }
    }
  }

  __device__ __forceinline__ static void load_chunk(T* sA, T* sB, const Mat<T>& a, const Mat<T>& b,
                                                    const int32_t* srow, int chunk, int m0, int n0,
                                                    int M, int N, int Kr, bool va, bool vb,
                                                    bool do_a = true, bool do_b = true) {
    const int k0 = chunk * KC;
    load_chunk_vec(sA, sB, a, b, srow, k0, m0, n0, M, N, Kr, va, vb, do_a, do_b);
    if (!va && do_a)
#pragma unroll 2
    for (int e = threadIdx.x; e < A_ELEMS; e += NT) {
      int kk, mm;
      if (AK) { kk = e % KC; mm = e / KC; } else { mm = e % BM; kk = e / BM; }
      const int k = k0 + kk, m = m0 + mm;
      const bool ok = (k < Kr) && (m < M);
      const T* g = a.base;
      if (ok) g = AK ? a.base + a_row(a, srow, m - 0) + k : a.base + a_row(a, srow, k) + m;
      T* s = AK ? sA + mm * A_LD + kk : sA + kk * A_LD + mm;
      cp_async<sizeof(T)>(s, g, ok);
    }
    if (!vb && do_b)
#pragma unroll 2
    for (int e = threadIdx.x; e < B_ELEMS; e += NT) {
      int kk, nn;
      if (BK) { kk = e % KC; nn = e / KC; } else { nn = e % BN; kk = e / BN; }
      const int k = k0 + kk, n = n0 + nn;
      const bool ok = (k < Kr) && (n < N);
      const T* g = b.base;
      if (ok) g = BK ? b.base + (int64_t)n * b.ld + k : b.base + (int64_t)k * b.ld + n;
      T* s = BK ? sB + nn * B_LD + kk : sB + kk * B_LD + nn;
      cp_async<sizeof(T)>(s, g, ok);
    }
  }

  // whether an operand may take the 16-byte path: aligned base, row pitch
  // and the extent of its contiguous dimension all multiples of VEC
  __device__ __forceinline__ static bool vec_ok(const Mat<T>& x, int contig_extent) {
    return ((reinterpret_cast<uintptr_t>(x.base) & 15) == 0) && (x.ld % VEC == 0) &&
           (contig_extent % VEC == 0);
  }

  // srow: gather indices for A's gathered dimension (m if AK, k otherwise),
  // staged in smem, indexed by absolute row.  CHECK_A: return whether any A
  // element of the tile is non-finite (block-wide).  COLSUM: threads t < BN
  // accumulate Σ_k B(k, n0+t) into *colsum, k ascending (the bias gradient).
  __device__ __forceinline__ static int run(T* smem, const Mat<T>& a, const Mat<T>& b,
                                            const int32_t* srow, int m0, int n0, int M, int N,
                                            int Kr, bool CHECK_A = false, T* colsum = nullptr,
                                            int c_lo = 0, int c_hi = -1, bool a_issued = false) {
    const bool COLSUM = colsum != nullptr;
    const bool va = vec_ok(a, AK ? Kr : M);
    const bool vb = vec_ok(b, BK ? Kr : N);
    const int slice = threadIdx.x / TPS, lt = threadIdx.x % TPS;
    const int tc = lt % CS, tr = lt / CS;
    T acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j] = T(0);
    bool bad = false;
    T csum = T(0);
    // chunks [c_lo, c_hi) of the k range (all of it by default); stage slots
    // follow the absolute chunk index
    const int nch = c_hi >= 0 ? c_hi : (Kr + KC - 1) / KC;
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      const int c = c_lo + s;
      if (c < nch)
        load_chunk(smem + (c % STAGES) * (A_STAGE + B_STAGE),
                   smem + (c % STAGES) * (A_STAGE + B_STAGE) + A_STAGE, a, b, srow, c, m0, n0, M,
                   N, Kr, va, vb, !a_issued, true);
      cp_commit();
    }
    for (int c = c_lo; c < nch; ++c) {
      const int pre = c + STAGES - 1;
      if (pre < nch) {
        T* st = smem + (pre % STAGES) * (A_STAGE + B_STAGE);
        load_chunk(st, st + A_STAGE, a, b, srow, pre, m0, n0, M, N, Kr, va, vb);
      }
      cp_commit();
      cp_wait<STAGES - 1>();
      __syncthreads();
      const T* sA = smem + (c % STAGES) * (A_STAGE + B_STAGE);
      const T* sB = sA + A_STAGE;
#pragma unroll 4
      for (int q = 0; q < KS; ++q) {
        const int kk = slice * KS + q;
        T av[TM], bv[TN];
#pragma unroll
        for (int i = 0; i < TM; ++i) {
          av[i] = AK ? sA[(tr + i * RS) * A_LD + kk] : sA[kk * A_LD + tr + i * RS];
          if (CHECK_A) bad |= !finite(av[i]);
        }
#pragma unroll
        for (int j = 0; j < TN; ++j)
          bv[j] = BK ? sB[(tc + j * CS) * B_LD + kk] : sB[kk * B_LD + tc + j * CS];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
      }
      if (COLSUM && threadIdx.x < BN) {
#pragma unroll 8
        for (int kk = 0; kk < KC; ++kk)
          csum += BK ? sB[threadIdx.x * B_LD + kk] : sB[kk * B_LD + threadIdx.x];
      }
      __syncthreads();
    }
    cp_wait<0>();
    if (COLSUM && threadIdx.x < BN) *colsum = csum;
    T* red = smem + slice * (BM * BN);
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) red[(tr + i * RS) * BN + tc + j * CS] = acc[i][j];
    return __syncthreads_or(bad);
  }

  // The prologue's A chunks alone (uncommitted: they join the first cp.async
  // group of run / run_seg called with a_issued).  For an A that does not
  // depend on the previous launch: issued before the PDL wait, B after it.
  __device__ static void prologue_a(T* smem, const Mat<T>& a, const int32_t* srow, int m0, int M,
                                    int Kr, int c_lo, int c_hi) {
    const bool va = vec_ok(a, AK ? Kr : M);
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      const int c = c_lo + s;
      if (c < c_hi)
        load_chunk(smem + (c % STAGES) * (A_STAGE + B_STAGE),
                   smem + (c % STAGES) * (A_STAGE + B_STAGE) + A_STAGE, a, a, srow, c, m0, 0, M,
                   0, Kr, va, false, true, false);
    }
  }

  // Input-range segmented variant (FWD split, fwd_tile): chunks [c_lo, c_hi)
  // in ranges of `cps` chunks aligned at multiples of cps.  At every range end
  // the slice partials go through `seg` (SK*BM*BN elements outside the
  // pipeline) and are reduced in value()'s order; thread t < BM*BN owns tile
  // element t.  part != nullptr: range r's tile is stored at part + r*BM*BN;
  // else the ranges are left-folded and the fold is left in seg[0, BM*BN).
  static constexpr int SEG = SK * BM * BN;
  __device__ static int run_seg(T* smem, T* seg, const Mat<T>& a, const Mat<T>& b,
                                const int32_t* srow, int m0, int n0, int M, int N, int Kr,
                                bool CHECK_A, int c_lo, int c_hi, int cps, T* part,
                                bool a_issued = false) {
    static_assert(BM * BN <= NT, "one tile element per thread");
    const bool va = vec_ok(a, AK ? Kr : M);
    const bool vb = vec_ok(b, BK ? Kr : N);
    const int slice = threadIdx.x / TPS, lt = threadIdx.x % TPS;
    const int tc = lt % CS, tr = lt / CS;
    T acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j] = T(0);
    bool bad = false;
    T fold = T(0);
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      const int c = c_lo + s;
      if (c < c_hi)
        load_chunk(smem + (c % STAGES) * (A_STAGE + B_STAGE),
                   smem + (c % STAGES) * (A_STAGE + B_STAGE) + A_STAGE, a, b, srow, c, m0, n0, M,
                   N, Kr, va, vb, !a_issued, true);
      cp_commit();
    }
    for (int c = c_lo; c < c_hi; ++c) {
      const int pre = c + STAGES - 1;
      if (pre < c_hi) {
        T* st = smem + (pre % STAGES) * (A_STAGE + B_STAGE);
        load_chunk(st, st + A_STAGE, a, b, srow, pre, m0, n0, M, N, Kr, va, vb);
      }
      cp_commit();
      cp_wait<STAGES - 1>();
      __syncthreads();
      const T* sA = smem + (c % STAGES) * (A_STAGE + B_STAGE);
      const T* sB = sA + A_STAGE;
#pragma unroll 4
      for (int q = 0; q < KS; ++q) {
        const int kk = slice * KS + q;
        T av[TM], bv[TN];
#pragma unroll
        for (int i = 0; i < TM; ++i) {
          av[i] = AK ? sA[(tr + i * RS) * A_LD + kk] : sA[kk * A_LD + tr + i * RS];
          if (CHECK_A) bad |= !finite(av[i]);
        }
#pragma unroll
        for (int j = 0; j < TN; ++j)
          bv[j] = BK ? sB[(tc + j * CS) * B_LD + kk] : sB[kk * B_LD + tc + j * CS];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
      }
      if (c + 1 == c_hi || (c + 1) % cps == 0) {  // range end
        T* red = seg + slice * (BM * BN);
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) {
            red[(tr + i * RS) * BN + tc + j * CS] = acc[i][j];
            acc[i][j] = T(0);
          }
        __syncthreads();
        if (threadIdx.x < BM * BN) {
          T v = seg[threadIdx.x];
#pragma unroll
          for (int s = 1; s < SK; ++s) v += seg[s * BM * BN + threadIdx.x];
          if (part) __stcg(part + (size_t)(c / cps) * (BM * BN) + threadIdx.x, v);
          else fold = (c / cps == c_lo / cps) ? v : fold + v;
        }
      }
      __syncthreads();
    }
    cp_wait<0>();
    if (!part && threadIdx.x < BM * BN) seg[threadIdx.x] = fold;
    return __syncthreads_or(bad);
  }

  __device__ __forceinline__ static T value(const T* smem, int mm, int nn) {
    T v = smem[mm * BN + nn];
#pragma unroll
    for (int s = 1; s < SK; ++s) v += smem[s * BM * BN + mm * BN + nn];
    return v;
  }
};

// tile shapes: fixed per tile kind (never per pack) → K-invariant
template <typename T> using FwdG = Gemm<T, 32, 8, 64, 4, 4, 16, 6, true, false>;
constexpr int FWD_KC = 64;  // FwdG's chunk
template <typename T> using TailG = Gemm<T, 16, 32, 64, 2, 4, 4, 4, true, false>;
template <typename T> using DgradG = Gemm<T, 32, 16, 64, 4, 4, 8, 4, true, true>;
template <typename T> using WgradG = Gemm<T, 32, 32, 32, 4, 4, 4, 4, false, false>;
// narrow layers (out <= 16): 64 x 16 tiles, the same 1024 elements per CTA
// and the same per-element sums (chunk / slice order), half the CTAs
template <typename T> using WgradNG = Gemm<T, 64, 16, 32, 8, 2, 4, 4, false, false>;
constexpr int WGN_BM = 64, WGN_BN = 16;
constexpr int FWD_BM = 32, FWD_BN = 8;
// TAIL: 16-row tiles — its serial softmax-xent + dgrad chain is per row, so
// small batches spread over more CTAs (the per-element sums are unchanged)
constexpr int TAIL_BM = 16, TAIL_MAXC = 32;
constexpr int HEAD_BM = 32;
constexpr int DG_BM = 32, DG_BN = 16;
constexpr int WG_BM = 32, WG_BN = 32;

// smem (bytes) a tile kind needs besides the GEMM pipeline
template <typename T>
struct Smem {
  static constexpr int ROWS = ROWCAP * 4;
  static constexpr int FWD = (FwdG<T>::SMEM_T + FwdG<T>::SEG) * (int)sizeof(T) + ROWS;
  static constexpr int WGRAD = (WgradG<T>::SMEM_T > WgradNG<T>::SMEM_T ? WgradG<T>::SMEM_T
                                                                       : WgradNG<T>::SMEM_T) *
                                   (int)sizeof(T) + ROWS;
  static constexpr int DGRAD = DgradG<T>::SMEM_T * (int)sizeof(T);
  static constexpr int HEAD = ROWS;
  // TAIL: pipeline + resident W_L [in x C] + dZ block [32 x 33] + rows
  __host__ __device__ static int tail(int in, int C) {
    return TailG<T>::SMEM_T * (int)sizeof(T) + in * C * (int)sizeof(T) +
           TAIL_BM * (TAIL_MAXC + 1) * (int)sizeof(T) + ROWS + TAIL_BM * 4;
  }
};

__device__ __forceinline__ void flag_min(int32_t* p, int v) { atomicMin(p, v); }

template <typename T>
__device__ __forceinline__ int64_t feed_row(const FeedDev<T>& f, int r) {
  return f.rows ? (int64_t)f.rows[r] : f.row0 + r;
}

// cache the batch's gather indices (rows [0, n)) in shared memory
template <typename T>
__device__ __forceinline__ void stage_rows(int32_t* srow, const FeedDev<T>& f, int n) {
  n = n < ROWCAP ? n : ROWCAP;
  for (int r = threadIdx.x; r < n; r += NT) srow[r] = (int32_t)feed_row(f, r);
}

template <typename T>
__device__ __forceinline__ Mat<T> input_mat(const MemberDev<T>& M, const FeedDev<T>& f, int l) {
  if (l == 0) return Mat<T>{f.feat, f.rows, f.row0, f.ld};
  return Mat<T>{M.A[l - 1], nullptr, 0, M.dims[l]};
}

// ---------------------------------------------------------------- FWD --
// Input-range split (pk_pack.cuh emit): a member whose layer input spans
// more than two chunks reduces it in fixed ranges of `cps` chunks (from its
// shape alone), each range's partial tile reduced separately and the ranges
// left-folded in order — so its arithmetic is the same however many CTAs
// share a tile (packed == standalone bitwise).  When the phase leaves SMs
// idle (small batch / narrow layer: the per-chunk latency chain of one CTA
// dominates) a tile gets ng CTAs, CTA g owning ranges [g*R/ng, (g+1)*R/ng);
// they store their range tiles in the pack workspace and the last to arrive
// folds them and runs the epilogue.  Tile bits: n0 [0,20) column, [20,27)
// cps (0 = unsplit); m0 [0,20) row, [20,24) g, [24,28) ng - 1.
constexpr int kFwdMaxRanges = 8;
__host__ __device__ inline int fwd_tile_n0(int32_t v) { return v & 0xFFFFF; }
__host__ __device__ inline int fwd_tile_m0(int32_t v) { return v & 0xFFFFF; }
__host__ __device__ inline int32_t fwd_pack_n0(int n0, int cps) { return n0 | (cps << 20); }
__host__ __device__ inline int32_t fwd_pack_m0(int m0, int g, int ng) {
  return m0 | (g << 20) | ((ng - 1) << 24);
}

template <typename T>
__device__ __noinline__ void prefetch_params(const PhaseArgs<T>& P);

template <typename T>
__device__ void fwd_tile(char* sm, const MemberDev<T>& M, const FeedDev<T>& f, const Tile& t,
                         int32_t* ws, const PhaseArgs<T>* first = nullptr) {
  using G = FwdG<T>;
  const int l = t.layer, in = M.dims[l], out = M.dims[l + 1];
  const int n0 = fwd_tile_n0(t.n0), m0 = fwd_tile_m0(t.m0), cps = (t.n0 >> 20) & 127;
  const int g = (t.m0 >> 20) & 15, ng = ((t.m0 >> 24) & 15) + 1;
  const int nch = (in + FWD_KC - 1) / FWD_KC;
  const int NR = cps ? (nch + cps - 1) / cps : 1;
  const int r_lo = g * NR / ng, r_hi = (g + 1) * NR / ng;
  const int R = f.take;
  T* smem = reinterpret_cast<T*>(sm);
  T* seg = smem + G::SMEM_T;
  int32_t* srow = reinterpret_cast<int32_t*>(sm + (G::SMEM_T + G::SEG) * sizeof(T));
  const Mat<T> a = input_mat(M, f, l);
  if (l == 0) stage_rows(srow, f, R);
  if (l > 0) pdl_wait();  // A_{l-1} comes from the previous phase
  __syncthreads();
  if (first) {
    // the step's first launch (k_phase): the batch rows do not depend on the
    // previous step, so their first chunks load before the PDL wait; the
    // parity, halt flag and parameters are read after it
    G::prologue_a(smem, a, srow, m0, R, in, cps ? r_lo * cps : 0,
                  cps ? min(nch, r_hi * cps) : nch);
    pdl_wait();
    pdl_launch();
    if (halted(*first)) {
      cp_commit();
      cp_wait<0>();
      return;
    }
    if (first->prefetch) prefetch_params(*first);
  }
  const int par = M.ctl->parity;
  const T* W = M.params[par] + M.w_off[l];
  const T* bias = M.params[par] + M.b_off[l];
  const Mat<T> b{W, nullptr, 0, out};
  constexpr int TS = FWD_BM * FWD_BN;
  static_assert(TS == NT, "one tile element per thread in the epilogue");
  // the thread's bias element, fetched under the GEMM
  const T bias_e = (n0 + (int)threadIdx.x % FWD_BN < out) ? bias[n0 + threadIdx.x % FWD_BN] : T(0);
  // workspace (pk_pack: d_done): [4 ints][one counter per CTA][8 range tiles per CTA]
  const int b0 = blockIdx.x - g;
  T* part = ng > 1 ? reinterpret_cast<T*>(ws + 4 + ((gridDim.x + 3) & ~3u)) +
                         (size_t)b0 * kFwdMaxRanges * TS
                   : nullptr;
  // layer 0: the input node's finite check (engine.py:233-235) rides on the
  // A operand already staged in shared memory
  PK_TRACE(1);
  int badx;
  const bool ai = first != nullptr;
  if (cps)
    badx = G::run_seg(smem, seg, a, b, srow, m0, n0, R, out, in, l == 0, r_lo * cps,
                      min(nch, r_hi * cps), cps, part, ai);
  else
    badx = (l == 0) ? G::run(smem, a, b, srow, m0, n0, R, out, in, true, nullptr, 0, -1, ai)
                    : G::run(smem, a, b, srow, m0, n0, R, out, in, false, nullptr, 0, -1, ai);
  PK_TRACE(2);
  const bool last = (l == M.n_layers - 1);
  int bad = badx ? 0 : INT_MAX;
  if (part) {
    __threadfence();
    __shared__ int arrived_last;
    __syncthreads();
    if (threadIdx.x == 0)
      arrived_last = (atomicAdd(ws + 4 + b0, r_hi - r_lo) + (r_hi - r_lo) == NR);
    __syncthreads();
    if (!arrived_last) {
      if (badx && threadIdx.x == 0) flag_min(&M.ctl->bad_node, 0);
      return;
    }
    __threadfence();
    if (threadIdx.x == 0) ws[4 + b0] = 0;  // ready for the next launch
    if (threadIdx.x < TS) {  // all range tiles in flight at once, then the fold
      T pv[kFwdMaxRanges];
#pragma unroll
      for (int r = 0; r < kFwdMaxRanges; ++r)
        pv[r] = r < NR ? __ldcg(part + (size_t)r * TS + threadIdx.x) : T(0);
      T v = pv[0];
#pragma unroll
      for (int r = 1; r < kFwdMaxRanges; ++r)
        if (r < NR) v += pv[r];
      seg[threadIdx.x] = v;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < FWD_BM * FWD_BN; e += NT) {
    const int mm = e / FWD_BN, nn = e % FWD_BN;
    const int m = m0 + mm, n = n0 + nn;
    if (m >= R || n >= out) continue;
    const T acc = cps ? seg[e] : G::value(smem, mm, nn);
    const T z = acc + bias_e;
    M.Z[l][(int64_t)m * out + n] = z;
    if (!finite(z)) bad = min(bad, 1 + 2 * l);
    if (!last) {
      const T av = act_fwd(M.act, z);
      M.A[l][(int64_t)m * out + n] = av;
      if (!finite(av)) bad = min(bad, 2 + 2 * l);
    }
  }
  if (bad != INT_MAX) flag_min(&M.ctl->bad_node, bad);
}

// ------------------------------------------------------- softmax-xent --
// One warp per row (lanes over classes): loss term −logp[y] into rowloss,
// dlogits = (p − onehot(y)) / R (engine.py:211-230, :252-264).
template <typename T>
__device__ __forceinline__ void xent_row(const T* z, T* dz, int C, int y, int R, bool train,
                                         double* rowloss) {
  const int lane = threadIdx.x & 31;
  T mx = -INFINITY;
  for (int c = lane; c < C; c += 32) mx = max(mx, z[c]);
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  T s = T(0);
  for (int c = lane; c < C; c += 32) s += ex(z[c] - mx);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const T zy = z[y];  // before dz (which may alias z) is written
  __syncwarp();
  if (train) {
    const T inv = T(1) / s, nv = T(R);
    for (int c = lane; c < C; c += 32) {
      T p = ex(z[c] - mx) * inv;
      if (c == y) p -= T(1);
      dz[c] = p / nv;
    }
  }
  if (lane == 0 && rowloss) *rowloss = -(double)((zy - mx) - lg(s));
}

// xent_row for C <= 16 on a half warp (lanes [16h, 16h+16)): the same
// butterfly minus its first step, which only folds in the idle lanes' -inf /
// 0 — identical results.  Both halves run the shuffles; `active` gates the
// row's reads and writes.
template <typename T>
__device__ __forceinline__ void xent_row16(const T* z, T* dz, int C, int y, int R, bool train,
                                           double* rowloss, bool active) {
  const int lane = threadIdx.x & 15;
  T mx = -INFINITY;
  if (active && lane < C) mx = z[lane];
#pragma unroll
  for (int o = 8; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o, 16));
  T s = T(0);
  if (active && lane < C) s = ex(z[lane] - mx);
#pragma unroll
  for (int o = 8; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, 16);
  const T zy = active ? z[y] : T(0);  // before dz (which may alias z) is written
  __syncwarp();
  if (!active) return;
  if (train && lane < C) {
    const T inv = T(1) / s, nv = T(R);
    T p = ex(z[lane] - mx) * inv;
    if (lane == y) p -= T(1);
    dz[lane] = p / nv;
  }
  if (lane == 0 && rowloss) *rowloss = -(double)((zy - mx) - lg(s));
}

template <typename T>
__device__ void head_tile(char* sm, const MemberDev<T>& M, const FeedDev<T>& f, const Tile& t,
                          bool train) {
  const int L = M.n_layers - 1, C = M.dims[L + 1];
  const int R = f.take;
  int32_t* ylab = reinterpret_cast<int32_t*>(sm);
  if (threadIdx.x < HEAD_BM && t.m0 + (int)threadIdx.x < R)
    ylab[threadIdx.x] = f.labels[feed_row(f, t.m0 + threadIdx.x)];
  pdl_wait();
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  for (int mm = warp; mm < HEAD_BM && t.m0 + mm < R; mm += NT / 32) {
    const int r = t.m0 + mm;
    xent_row(M.Z[L] + (int64_t)r * C, M.dZ[L] + (int64_t)r * C, C, ylab[mm], R, train,
             M.rowloss + r);
  }
}

// --------------------------------------------------------------- TAIL --
template <typename T>
__device__ void tail_tile(char* sm, const MemberDev<T>& M, const FeedDev<T>& f, const Tile& t,
                          bool train) {
  using G = TailG<T>;
  const int L = M.n_layers - 1, in = M.dims[L], C = M.dims[L + 1];
  const int R = f.take;
  T* smem = reinterpret_cast<T*>(sm);
  T* sW = smem + G::SMEM_T;                 // W_L [in][C]
  T* sD = sW + in * C;                      // logits → dlogits block [32][TAIL_MAXC+1]
  int32_t* srow = reinterpret_cast<int32_t*>(sD + TAIL_BM * (TAIL_MAXC + 1));
  int32_t* ylab = srow + ROWCAP;            // labels of the block's rows
  const int par = M.ctl->parity;
  const T* W = M.params[par] + M.w_off[L];
  const T* bias = M.params[par] + M.b_off[L];
  // parameters and labels do not depend on the previous phase: fetch them
  // before waiting on it
  const bool dgrad = train && L > 0;
  if (dgrad) {
    for (int e = threadIdx.x; e < in * C; e += NT) cp_async<sizeof(T)>(sW + e, W + e, true);
    cp_commit();
  }
  if (threadIdx.x < TAIL_BM && t.m0 + (int)threadIdx.x < R)
    ylab[threadIdx.x] = f.labels[feed_row(f, t.m0 + threadIdx.x)];
  // the thread's bias element (its column is fixed: NT is a multiple of TAIL_MAXC)
  static_assert(NT % TAIL_MAXC == 0, "fixed epilogue column per thread");
  const int ce = threadIdx.x % TAIL_MAXC;
  const T bias_e = ce < C ? bias[ce] : T(0);
  if (L == 0) stage_rows(srow, f, R);
  if (L > 0) pdl_wait();
  __syncthreads();
  const Mat<T> a = input_mat(M, f, L);
  const Mat<T> b{W, nullptr, 0, C};
  PK_TRACE(1);
  const int badx = (L == 0) ? G::run(smem, a, b, srow, t.m0, 0, R, C, in, true)
                            : G::run(smem, a, b, srow, t.m0, 0, R, C, in, false);
  PK_TRACE(2);
  int bad = badx ? 0 : INT_MAX;
  for (int e = threadIdx.x; e < TAIL_BM * TAIL_MAXC; e += NT) {
    const int mm = e / TAIL_MAXC, c = e % TAIL_MAXC;
    const int m = t.m0 + mm;
    if (m >= R || c >= C) continue;
    const T z = G::value(smem, mm, c) + bias_e;
    M.Z[L][(int64_t)m * C + c] = z;
    sD[mm * (TAIL_MAXC + 1) + c] = z;
    if (!finite(z)) bad = min(bad, 1 + 2 * L);
  }
  if (bad != INT_MAX) flag_min(&M.ctl->bad_node, bad);
  __syncthreads();
  // softmax-xent per row, in place in sD (logits → dlogits)
  const int warp = threadIdx.x >> 5;
  if (C <= 16) {  // two rows per warp
    for (int m2 = 2 * warp; m2 < TAIL_BM && t.m0 + m2 < R; m2 += NT / 16) {
      const int mm = m2 + ((threadIdx.x >> 4) & 1);
      const bool act = mm < TAIL_BM && t.m0 + mm < R;
      T* row = sD + (act ? mm : m2) * (TAIL_MAXC + 1);
      xent_row16(row, row, C, act ? ylab[mm] : 0, R, train, M.rowloss + t.m0 + mm, act);
    }
  } else {
    for (int mm = warp; mm < TAIL_BM && t.m0 + mm < R; mm += NT / 32) {
      T* row = sD + mm * (TAIL_MAXC + 1);
      xent_row(row, row, C, ylab[mm], R, train, M.rowloss + t.m0 + mm);
    }
  }
  PK_TRACE(3);
  if (!train) return;
  __syncthreads();
  for (int e = threadIdx.x; e < TAIL_BM * C; e += NT) {
    const int mm = e / C, c = e % C;
    if (t.m0 + mm < R) M.dZ[L][(int64_t)(t.m0 + mm) * C + c] = sD[mm * (TAIL_MAXC + 1) + c];
  }
  if (!dgrad) return;
  cp_wait<0>();
  __syncthreads();
  PK_TRACE(4);
  // dZ_{L-1}[m][i] = act'(Z,A)[m][i] · Σ_c dZ_L[m][c] W_L[i][c]; the Z/A
  // operands of a batch of outputs are loaded before any is computed
  const T* __restrict__ Zp = M.Z[L - 1];
  const T* __restrict__ Ap = M.A[L - 1];
  T* __restrict__ dZp = M.dZ[L - 1];
  const int rows = min(TAIL_BM, R - t.m0);
  const int total = rows * in;
  constexpr int B8 = 8;
  for (int e0 = 0; e0 < total; e0 += NT * B8) {
    T zv[B8], avv[B8];
#pragma unroll
    for (int u = 0; u < B8; ++u) {
      const int e = e0 + u * NT + threadIdx.x;
      if (e < total) {
        const int64_t o = (int64_t)(t.m0 + e / in) * in + e % in;
        zv[u] = Zp[o];
        avv[u] = Ap[o];
      }
    }
#pragma unroll
    for (int u = 0; u < B8; ++u) {
      const int e = e0 + u * NT + threadIdx.x;
      if (e >= total) break;
      const int mm = e / in, i = e % in;
      const T* d = sD + mm * (TAIL_MAXC + 1);
      const T* w = sW + i * C;
      T s = T(0);
      for (int c = 0; c < C; ++c) s = fma(d[c], w[c], s);
      dZp[(int64_t)(t.m0 + mm) * in + i] = act_bwd(M.act, zv[u], avv[u], s);
    }
  }
}

// -------------------------------------------------------------- DGRAD --
template <typename T>
__device__ void dgrad_tile(char* sm, const MemberDev<T>& M, const FeedDev<T>& f, const Tile& t) {
  using G = DgradG<T>;
  const int l = t.layer, in = M.dims[l], out = M.dims[l + 1];
  const int R = f.take;
  T* smem = reinterpret_cast<T*>(sm);
  const int par = M.ctl->parity;
  const T* W = M.params[par] + M.w_off[l];
  pdl_wait();
  const Mat<T> a{M.dZ[l], nullptr, 0, out};
  const Mat<T> b{W, nullptr, 0, out};  // B(k=j, n=i) = W[i][j]
  G::run(smem, a, b, nullptr, t.m0, t.n0, R, in, out);
  constexpr int PER = DG_BM * DG_BN / NT;
  T zv[PER], avv[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int e = u * NT + threadIdx.x;
    const int m = t.m0 + e / DG_BN, n = t.n0 + e % DG_BN;
    if (m < R && n < in) {
      zv[u] = M.Z[l - 1][(int64_t)m * in + n];
      avv[u] = M.A[l - 1][(int64_t)m * in + n];
    }
  }
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int e = u * NT + threadIdx.x;
    const int mm = e / DG_BN, nn = e % DG_BN;
    const int m = t.m0 + mm, n = t.n0 + nn;
    if (m < R && n < in)
      M.dZ[l - 1][(int64_t)m * in + n] = act_bwd(M.act, zv[u], avv[u], G::value(smem, mm, nn));
  }
}

// -------------------------------------------------------------- WGRAD --
template <typename T, int WB>
__device__ void wgrad_tile(char* sm, const MemberDev<T>& M, const FeedDev<T>& f, const Tile& t) {
  using G = typename std::conditional<WB == WGN_BM, WgradNG<T>, WgradG<T>>::type;
  constexpr int WG_BM = WB, WG_BN = WB == WGN_BM ? WGN_BN : 32;
  const int l = t.layer, in = M.dims[l], out = M.dims[l + 1];
  const int R = f.take;
  T* smem = reinterpret_cast<T*>(sm);
  int32_t* srow = reinterpret_cast<int32_t*>(sm + G::SMEM_T * sizeof(T));
  const MemberCtl* ctl = M.ctl;
  const int par = ctl->parity;
  const int64_t P = M.s_stride;  // slot block stride
  const T* __restrict__ wc = M.params[par];
  T* __restrict__ wn = M.params[par ^ 1];
  const T* sc = M.slots[par];
  T* sn = M.slots[par ^ 1];
  // pull this tile's weights + slots toward L2 while the previous phase drains
  if ((int)threadIdx.x < WG_BM && t.m0 + (int)threadIdx.x < in) {
    const int64_t row = M.w_off[l] + (int64_t)(t.m0 + threadIdx.x) * out + t.n0;
    const int cnt = min(WG_BN, out - t.n0);
    for (int s = -1; s < M.n_slots; ++s) {
      const T* base = s < 0 ? wc : sc + (int64_t)s * P;
      const uintptr_t p0 = reinterpret_cast<uintptr_t>(base + row) & ~(uintptr_t)15;
      const uintptr_t p1 = reinterpret_cast<uintptr_t>(base + row + cnt);
      l2_prefetch_lines(reinterpret_cast<const void*>(p0), (uint32_t)(p1 - p0));
    }
  }
  const T* __restrict__ s0c = sc;
  T* __restrict__ s0n = sn;
  const T* __restrict__ s1c = sc ? sc + P : nullptr;
  T* __restrict__ s1n = sn ? sn + P : nullptr;
  // optimizer operands: every element's weight and slots are gathered before
  // the GEMM (they do not depend on earlier phases; one round trip per
  // tensor, hidden under the GEMM — the L2 prefetch above warmed them)
  constexpr int PER = WG_BM * WG_BN / NT;
  int64_t idx[PER];
  bool ok[PER];
  T w[PER], s0[PER], s1[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int e = u * NT + threadIdx.x;
    const int m = t.m0 + e / WG_BN, n = t.n0 + e % WG_BN;
    ok[u] = (m < in && n < out);
    idx[u] = M.w_off[l] + (int64_t)m * out + n;
    if (ok[u]) {
      w[u] = wc[idx[u]];
      if (M.n_slots >= 1) s0[u] = s0c[idx[u]];
      if (M.n_slots >= 2) s1[u] = s1c[idx[u]];
    }
  }
  const T lr = T(ctl->lr), wd = T(M.wd);
  T bc1 = T(1), bc2 = T(1);
  if (M.opt == PK_OPT_ADAM) {
    bc1 = T(ctl->bc1);
    bc2 = T(ctl->bc2);
  }
  const int gpos = 2 * (M.n_layers - 1 - l);
  const int fault = ctl->fault_grad;
  // layer 0: the input rows do not come from this step's launches — their
  // first chunks load before the PDL wait (inside G::run), dZ_0's after it
  // A(m=i, k=r) = input[r][i]; B(k=r, n=j) = dZ_l[r][j]; tiles on the first
  // row block also sum dZ_l's columns (the bias gradient) from the staged B
  const Mat<T> a = input_mat(M, f, l);
  const Mat<T> b{M.dZ[l], nullptr, 0, out};
  if (l == 0) {
    stage_rows(srow, f, R);
    __syncthreads();
    G::prologue_a(smem, a, srow, t.m0, in, R, 0, (R + G::KCH - 1) / G::KCH);
  }
  pdl_wait();
  __syncthreads();
  T gb = T(0);
  PK_TRACE(1);
  G::run(smem, a, b, srow, t.m0, t.n0, in, out, R, false, t.m0 == 0 ? &gb : nullptr, 0, -1,
         l == 0);
  PK_TRACE(2);
  bool badW = false;
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    if (!ok[u]) continue;
    const int e = u * NT + threadIdx.x;
    T g = G::value(smem, e / WG_BN, e % WG_BN);
    if (fault == gpos) g = T(NAN);
    badW |= !finite(g);
    opt_step(M.opt, lr, wd, bc1, bc2, w[u], s0[u], s1[u], g);
    wn[idx[u]] = w[u];
    if (M.n_slots >= 1) s0n[idx[u]] = s0[u];
    if (M.n_slots >= 2) s1n[idx[u]] = s1[u];
  }
  bool badB = false;
  if (t.m0 == 0 && (int)threadIdx.x < WG_BN && t.n0 + (int)threadIdx.x < out) {
    const int64_t i = M.b_off[l] + t.n0 + threadIdx.x;
    if (fault == gpos + 1) gb = T(NAN);
    badB = !finite(gb);
    T bw = wc[i], b0 = M.n_slots >= 1 ? s0c[i] : T(0), b1 = M.n_slots >= 2 ? s1c[i] : T(0);
    opt_step(M.opt, lr, wd, bc1, bc2, bw, b0, b1, gb);
    wn[i] = bw;
    if (M.n_slots >= 1) s0n[i] = b0;
    if (M.n_slots >= 2) s1n[i] = b1;
  }
  if (badW) flag_min(&M.ctl->bad_grad, gpos);
  if (badB) flag_min(&M.ctl->bad_grad, gpos + 1);
}

// ----------------------------------------------------------- FINALIZE --
// Run by the last CTA of the last phase.  Loss = Σ rowloss / R in a fixed
// order (thread-strided, fixed tree); commit rules of packing.py:246-253: a
// forward non-finite value aborts the step, else members commit in pack
// order until the first one with a non-finite gradient.
// FINALIZE for packs whose members all take the tensor path (two affine
// layers; loss and next Adam corrections already in ctl): one warp, lane =
// member, the same commit rules via ballots.
// a train step enqueued behind a failed one did no work: report it skipped,
// commit nothing (packed_run stops at the failed step's exception)
template <typename T>
__device__ __noinline__ void finalize_skipped(const PhaseArgs<T>& P) {
  int32_t* st = reinterpret_cast<int32_t*>(P.ring + (int64_t)hdr_of(P).slot * P.ring_stride);
  double* losses = reinterpret_cast<double*>(st + 4);
  for (int k = threadIdx.x; k < P.K; k += blockDim.x) losses[k] = 0.0;
  if (threadIdx.x == 0) {
    st[0] = PK_SKIPPED; st[1] = -1; st[2] = -1; st[3] = 0;
  }
}

template <typename T>
__device__ __noinline__ void finalize_fast(const PhaseArgs<T>& P) {
  if (threadIdx.x >= 32) return;
  const int K = P.K, k = threadIdx.x;
  MemberCtl* c = k < K ? P.ctl_in[k] : nullptr;
  const bool act = k < K && feed_of(P, k).take != 0;
  int bn = INT_MAX, bg = INT_MAX;
  double loss = 0.0;
  // every control-block field the commit reads, in one batch of loads (one
  // L2 round trip instead of two on the step's serial tail)
  int par = 0;
  int64_t steps = 0;
  double n1 = 0.0, n2 = 0.0;
  if (k < K) {
    bn = c->bad_node;
    bg = c->bad_grad;
    loss = c->loss;
    par = c->parity;
    steps = c->step_counter;
    n1 = c->bcn1;
    n2 = c->bcn2;
  }
  if (!act) bn = bg = INT_MAX;
  else if (!isfinite(loss)) bn = min(bn, 4);  // node 2·n_layers = the loss node
  int code = PK_OK, who = -1, idx = -1, stop = K;
  const unsigned mv = __ballot_sync(0xffffffffu, bn != INT_MAX);
  if (mv) {
    who = __ffs(mv) - 1;
    idx = __shfl_sync(0xffffffffu, bn, who);
    code = PK_ERR_NONFINITE_VALUE;
    stop = 0;
  } else {
    const unsigned mg = __ballot_sync(0xffffffffu, bg != INT_MAX);
    if (mg) {
      who = __ffs(mg) - 1;
      idx = __shfl_sync(0xffffffffu, bg, who);
      code = PK_ERR_NONFINITE_GRAD;
      stop = who;
    }
  }
  const bool commit = act && k < stop;
  const int committed = __popc(__ballot_sync(0xffffffffu, commit));
  int32_t* st = reinterpret_cast<int32_t*>(P.ring + (int64_t)hdr_of(P).slot * P.ring_stride);
  double* losses = reinterpret_cast<double*>(st + 4);
  if (k < K) {
    losses[k] = act ? loss : 0.0;
    if (commit) {
      c->parity = par ^ 1;
      c->step_counter = steps + 1;
      c->bc1 = n1;
      c->bc2 = n2;
    }
    if (act) c->fault_grad = -1;  // one-shot
    c->bad_node = INT_MAX;
    c->bad_grad = INT_MAX;
  }
  if (k == 0) {
    st[0] = code; st[1] = who; st[2] = idx; st[3] = committed;
    if (code != PK_OK && P.halt) *P.halt = 1;
  }
}

template <typename T>
__device__ __noinline__ void finalize(const PhaseArgs<T>& P, bool train) {
  __shared__ int s_bn[PK_MAX_PACK], s_bg[PK_MAX_PACK];
  __shared__ int s_code, s_who, s_idx, s_stop;
  const int K = P.K, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;  // kernels run 8 or 12 warps
  // K <= 32: the commit's operands (parity, step counter, Adam's next bias
  // corrections, the loss) are fetched / computed while the losses reduce —
  // by the last warp when it has no member to reduce, else by warp 0 — and
  // handed over in shared memory (no second round trip on the serial tail)
  __shared__ double f_loss[32], f_bc1[32], f_bc2[32];
  __shared__ long long f_step[32];
  __shared__ int f_par[32];
  const bool fast = train && K <= 32;
  if (fast && warp == (K < nw ? nw - 1 : 0) && lane < K && feed_of(P, lane).take) {
    const MemberDev<T>& M = P.mems[lane];
    const MemberCtl* c = M.ctl;
    const long long step = c->step_counter;
    f_par[lane] = c->parity;
    f_step[lane] = step;
    if (M.tensor) {
      f_bc1[lane] = c->bcn1;
      f_bc2[lane] = c->bcn2;
    } else if (M.opt == PK_OPT_ADAM) {
      adam_bias_corrections(step + 1, &f_bc1[lane], &f_bc2[lane]);
    }
  }
  // warp w reduces the loss terms of members w, w+8, ...: lane-strided
  // partial sums then a fixed butterfly (deterministic, K-invariant)
  for (int k = warp; k < K; k += nw) {
    const int take = feed_of(P, k).take;
    int bn = INT_MAX, bg = INT_MAX;
    if (take) {
      const MemberDev<T>& M = P.mems[k];
      MemberCtl* c = M.ctl;
      bn = c->bad_node;  // issued ahead of the row-loss loads
      bg = c->bad_grad;
      const double tl = (train && M.tensor) ? c->loss : 0.0;
      double s = 0.0;
      if (!(train && M.tensor)) {
        // four rows per lane in flight at once, summed in row order
        for (int r0 = lane; r0 < take; r0 += 128) {
          double x[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) x[u] = r0 + 32 * u < take ? M.rowloss[r0 + 32 * u] : 0.0;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (r0 + 32 * u < take) s += x[u];
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      }
      if (train) {
        const double loss = M.tensor ? tl : s / double(take);
        if (lane == 0) {
          c->loss = loss;
          if (fast) f_loss[k] = loss;
        }
        if (!isfinite(loss)) bn = min(bn, 2 * M.n_layers);
      } else if (lane == 0) {
        c->eval_acc += s;
      }
    }
    if (lane == 0) {
      s_bn[k] = bn;
      s_bg[k] = bg;
    }
  }
  PK_TRACE(8);
  __syncthreads();
  if (threadIdx.x == 0) {
    int code = PK_OK, who = -1, idx = -1, stop = K;
    for (int k = 0; k < K && train; ++k)
      if (s_bn[k] != INT_MAX) { code = PK_ERR_NONFINITE_VALUE; who = k; idx = s_bn[k]; stop = 0; break; }
    for (int k = 0; k < K && train && code == PK_OK; ++k)
      if (s_bg[k] != INT_MAX) { code = PK_ERR_NONFINITE_GRAD; who = k; idx = s_bg[k]; stop = k; }
    s_code = code; s_who = who; s_idx = idx; s_stop = stop;
  }
  __syncthreads();
  PK_TRACE(9);
  int32_t* st = reinterpret_cast<int32_t*>(P.ring + (int64_t)hdr_of(P).slot * P.ring_stride);
  double* losses = reinterpret_cast<double*>(st + 4);
  int committed = 0;
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    MemberCtl* c = P.mems[k].ctl;
    const bool act = feed_of(P, k).take != 0;
    if (train && fast) {
      losses[k] = act ? f_loss[k] : 0.0;
      if (act && k < s_stop) {
        c->parity = f_par[k] ^ 1;
        c->step_counter = f_step[k] + 1;
        if (P.mems[k].tensor || P.mems[k].opt == PK_OPT_ADAM) {  // the only reader: wgrad_tile
          c->bc1 = f_bc1[k];
          c->bc2 = f_bc2[k];
        }
        ++committed;
      }
      if (act) c->fault_grad = -1;  // one-shot
    } else if (train) {
      losses[k] = act ? c->loss : 0.0;
      if (act && k < s_stop) {
        c->parity ^= 1;
        c->step_counter += 1;
        if (P.mems[k].tensor) {
          c->bc1 = c->bcn1;
          c->bc2 = c->bcn2;
        } else if (P.mems[k].opt == PK_OPT_ADAM) {  // the only reader (wgrad_tile)
          adam_bias_corrections(c->step_counter, &c->bc1, &c->bc2);
        }
        ++committed;
      }
      if (act) c->fault_grad = -1;  // one-shot
    }
    c->bad_node = INT_MAX;
    c->bad_grad = INT_MAX;
  }
  PK_TRACE(10);
  committed = __syncthreads_count(committed > 0) ? committed : committed;
  __shared__ int s_comm;
  if (threadIdx.x == 0) s_comm = 0;
  __syncthreads();
  if (committed) atomicAdd(&s_comm, committed);
  __syncthreads();
  if (threadIdx.x == 0 && train) {
    st[0] = s_code; st[1] = s_who; st[2] = s_idx; st[3] = s_comm;
    if (s_code != PK_OK && P.halt) *P.halt = 1;
  }
}

// ------------------------------------------------------------- kernels --

// WGRAD tiles of narrow layers carry bit 20 of n0 (pk_pack.cuh emit)
__device__ __forceinline__ Tile wg_tile(Tile t) {
  t.n0 &= 0xFFFFF;
  return t;
}

// L2 prefetch of every active member's committed params + slots (first
// phase): the step's dominant HBM stream overlaps the forward pass.
template <typename T>
__device__ __noinline__ void prefetch_params(const PhaseArgs<T>& P) {
  constexpr uint32_t CH = 16384;
  const int64_t gt = (int64_t)blockIdx.x * NT + threadIdx.x;
  const int64_t gs = (int64_t)gridDim.x * NT;
  int64_t base = 0;
  for (int k = 0; k < P.K; ++k) {
    if (!feed_of(P, k).take) continue;
    const MemberDev<T>& M = P.mems[k];
    const int par = M.ctl->parity;
    for (int s = -1; s < M.n_slots; ++s) {
      // bulk prefetch needs 16-byte aligned address and size: round the
      // region out (slab regions are 256-byte padded, so this stays inside)
      const uintptr_t lo = reinterpret_cast<uintptr_t>(
          s < 0 ? M.params[par] : M.slots[par] + (int64_t)s * M.s_stride);
      const uintptr_t hi = lo + (uintptr_t)M.n_params * sizeof(T);
      const char* p = reinterpret_cast<const char*>(lo & ~(uintptr_t)15);
      const int64_t bytes = (int64_t)(((hi + 15) & ~(uintptr_t)15) - (lo & ~(uintptr_t)15));
      const int64_t nch = (bytes + CH - 1) / CH;
      for (int64_t c = (gt - base % gs + gs) % gs; c < nch; c += gs) {
        const int64_t off = c * CH;
        const int64_t left = bytes - off;
        l2_prefetch(p + off, (uint32_t)(left < (int64_t)CH ? left : (int64_t)CH));
      }
      base += nch;
    }
  }
}

// Common kernel tail: wait for the predecessor kernel (so kernels complete
// in stream order even for CTAs that had no dependent work), then the last
// CTA of the step's last launch runs FINALIZE.
template <typename T>
__device__ __forceinline__ void kernel_end(const PhaseArgs<T>& P, bool train) {
  PK_TRACE(5);
  pdl_wait();
  if (!P.is_last) return;
  __shared__ int last, was_halted;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    // the halt flag only changes in a FINALIZE (of an earlier step, complete
    // before this step's first launch passed its PDL wait): its load is
    // issued while the arrival atomic is in flight, not after it
    int prev, hv = 0;
    asm volatile("atom.add.gpu.global.u32 %0, [%1], 1;" : "=r"(prev) : "l"(P.done) : "memory");
    if (train && P.halt)
      asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(hv) : "l"(P.halt) : "memory");
    was_halted = hv != 0;
    last = (prev == (int)gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  PK_TRACE(6);
  if (train && was_halted) finalize_skipped<T>(P);
  else if (train && P.all_tensor) finalize_fast<T>(P);
  else finalize<T>(P, train);
  PK_TRACE(7);
  if (threadIdx.x == 0) *P.done = 0;
}

// Kind masks: one lean kernel per tile kind (plus WGRAD|DGRAD and a generic
// all-kinds kernel for mixed phases of ragged packs).  Keeping each kernel's
// code to the one path it runs keeps it resident in the SM instruction cache.
constexpr int KM_FWD = 1 << TK_FWD, KM_TAIL = 1 << TK_TAIL, KM_HEAD = 1 << TK_HEAD;
constexpr int KM_DGRAD = 1 << TK_DGRAD, KM_WGRAD = 1 << TK_WGRAD, KM_ALL = 31;

template <typename T, int MASK>
__global__ void __launch_bounds__(NT, 1) k_phase(const __grid_constant__ PhaseArgs<T> P) {
  extern __shared__ __align__(16) char smem_raw[];
  if (threadIdx.x == 0)
    pk_trace_slots = P.trace ? P.trace + (size_t)blockIdx.x * kTraceSlots : nullptr;
  PK_TRACE(0);
  // tiles, feeds and the step header are static or step-inline: readable
  // before the PDL wait
  const Tile t = tile_of(P);
  const FeedDev<T> f = feed_of(P, t.member);
  const bool train = (hdr_of(P).mode == 0);
  // a first-launch layer-0 FWD tile waits inside fwd_tile, after its batch
  // rows are in flight
  const bool early = (MASK & KM_FWD) && P.first && t.kind == TK_FWD && t.layer == 0 &&
                     f.take != 0 && fwd_tile_m0(t.m0) < f.take;
  if (early) {
    fwd_tile<T>(smem_raw, P.mems[t.member], f, t, P.done, &P);
    kernel_end(P, train);
    return;
  }
  pdl_begin(P);
  if (P.prefetch) prefetch_params(P);
  if (f.take != 0 && !halted(P)) {
    const MemberDev<T>& M = P.mems[t.member];
    if ((MASK & KM_FWD) && t.kind == TK_FWD) {
      if (fwd_tile_m0(t.m0) < f.take) fwd_tile<T>(smem_raw, M, f, t, P.done);
    } else if ((MASK & KM_TAIL) && t.kind == TK_TAIL) {
      if (t.m0 < f.take) tail_tile<T>(smem_raw, M, f, t, train);
    } else if ((MASK & KM_HEAD) && t.kind == TK_HEAD) {
      if (t.m0 < f.take) head_tile<T>(smem_raw, M, f, t, train);
    } else if ((MASK & KM_DGRAD) && t.kind == TK_DGRAD) {
      if (t.m0 < f.take) dgrad_tile<T>(smem_raw, M, f, t);
    } else if ((MASK & KM_WGRAD) && t.kind == TK_WGRAD) {
      if (t.n0 >> 20) wgrad_tile<T, WGN_BM>(smem_raw, M, f, wg_tile(t));
      else wgrad_tile<T, WG_BM>(smem_raw, M, f, t);
    }
  }
  kernel_end(P, train);
}

#include "pk_mlp1.cuh"
#include "pk_umma.cuh"
#include "pk_m1t.cuh"

// tcgen05 3xTF32 one-hidden-layer step (fp32 members only; the f64 device
// mode never schedules these phases)
template <typename T>
__global__ void __launch_bounds__(NT, 1) k_m1t_fwd(const __grid_constant__ PhaseArgs<T> P) {
  extern __shared__ __align__(128) char smem_raw[];
  if (threadIdx.x == 0)
    pk_trace_slots = P.trace ? P.trace + (size_t)blockIdx.x * kTraceSlots : nullptr;
  PK_TRACE(0);
  if (!P.first) pdl_launch();  // a step's first launch waits inside the tile (after its
                               // independent prologue) and releases its dependents then
  if constexpr (sizeof(T) == 4) {
    const Tile t = tile_of(P);
    const FeedDev<T> f = feed_of(P, t.member);
    first_touch(P, reinterpret_cast<const MemberDev<T>*>(mem_of(P, t.member)), f);
    // the member's descriptor in shared memory: every field read is an LDS,
    // not a global load on the critical path
    __shared__ MemberDev<float> sM;
    if (threadIdx.x < sizeof(MemberDev<float>) / 4)
      reinterpret_cast<int32_t*>(&sM)[threadIdx.x] =
          reinterpret_cast<const int32_t*>(mem_of(P, t.member))[threadIdx.x];
    __syncthreads();
    if (f.take != 0) {
      m1t_fwd_tile(smem_raw, sM, f, t.m0, t.n0, P.cs, P);
    } else if (P.first) {
      pdl_wait();
      pdl_launch();
    }
  } else {
    __trap();
  }
  kernel_end(P, true);
}

#include "pk_m1x.cuh"

// the whole one-hidden-layer step in one launch: a cluster of P.cs CTAs per
// member (fp32; members with batch <= 64, pk_m1x.cuh)
template <typename T>
__global__ void __launch_bounds__(NT, 1) k_m1x_step(const __grid_constant__ PhaseArgs<T> P) {
  extern __shared__ __align__(128) char smem_raw[];
  if (threadIdx.x == 0)
    pk_trace_slots = P.trace ? P.trace + (size_t)blockIdx.x * kTraceSlots : nullptr;
  PK_TRACE(0);
  pdl_begin(P);
  if constexpr (sizeof(T) == 4) {
    const Tile t = tile_of(P);
    const FeedDev<T> f = feed_of(P, t.member);
    __shared__ MemberDev<float> sM;
    if (threadIdx.x < sizeof(MemberDev<float>) / 4)
      reinterpret_cast<int32_t*>(&sM)[threadIdx.x] =
          reinterpret_cast<const int32_t*>(mem_of(P, t.member))[threadIdx.x];
    __syncthreads();
    // m0 = cluster rank (own unit range), layer = 16-unit blocks per CTA;
    // take and halt are uniform over the member's cluster
    if (f.take != 0 && !halted(P)) m1x_step(smem_raw, sM, f, t.m0, t.layer, P.stages);
  } else {
    __trap();
  }
  kernel_end(P, true);
}

template <typename T>
__global__ void __launch_bounds__(NT, 1) k_m1s_fwd(const __grid_constant__ PhaseArgs<T> P) {
  extern __shared__ __align__(128) char smem_raw[];
  if (threadIdx.x == 0)
    pk_trace_slots = P.trace ? P.trace + (size_t)blockIdx.x * kTraceSlots : nullptr;
  PK_TRACE(0);
  pdl_begin(P);
  if constexpr (sizeof(T) == 4) {
    const Tile t = tile_of(P);
    const FeedDev<T> f = feed_of(P, t.member);
    first_touch(P, reinterpret_cast<const MemberDev<T>*>(mem_of(P, t.member)), f);
    __shared__ MemberDev<float> sM;
    if (threadIdx.x < sizeof(MemberDev<float>) / 4)
      reinterpret_cast<int32_t*>(&sM)[threadIdx.x] =
          reinterpret_cast<const int32_t*>(mem_of(P, t.member))[threadIdx.x];
    __syncthreads();
    if (f.take != 0 && !halted(P)) {
      if (m1_rows_pad(sM.max_rows) == 32 && t_nsplit(sM.dims[0]) * 32 <= 512)
        m1s_fwd_tile_ws(smem_raw, sM, f, t.m0);
      else
        m1s_fwd_tile(smem_raw, sM, f, t.m0);
    }
  } else {
    __trap();
  }
  kernel_end(P, true);
}

template <typename T>
__global__ void __launch_bounds__(NT, 1) k_m1c_fwd(const __grid_constant__ PhaseArgs<T> P) {
  extern __shared__ __align__(128) char smem_raw[];
  if (threadIdx.x == 0)
    pk_trace_slots = P.trace ? P.trace + (size_t)blockIdx.x * kTraceSlots : nullptr;
  PK_TRACE(0);
  if (!P.first) pdl_launch();  // a first launch waits inside the tile, after its prologue
  if constexpr (sizeof(T) == 4) {
    const Tile t = tile_of(P);
    const FeedDev<T> f = feed_of(P, t.member);
    first_touch(P, reinterpret_cast<const MemberDev<T>*>(mem_of(P, t.member)), f);
    __shared__ MemberDev<float> sM;
    if (threadIdx.x < sizeof(MemberDev<float>) / 4)
      reinterpret_cast<int32_t*>(&sM)[threadIdx.x] =
          reinterpret_cast<const int32_t*>(mem_of(P, t.member))[threadIdx.x];
    __syncthreads();
    // m0 = unit tile, n0 = cluster rank (input-split range)
    if (f.take != 0) {
      m1c_fwd_tile(smem_raw, sM, f, t.m0, t.n0, P.cs, P);
    } else if (P.first) {
      pdl_wait();
      pdl_launch();
    }
  } else {
    __trap();
  }
  kernel_end(P, true);
}

template <typename T>
__global__ void __launch_bounds__(T_BWD_NT, 1) k_m1t_bwd(const __grid_constant__ PhaseArgs<T> P) {
  extern __shared__ __align__(128) char smem_raw[];
  if (threadIdx.x == 0)
    pk_trace_slots = P.trace ? P.trace + (size_t)blockIdx.x * kTraceSlots : nullptr;
  PK_TRACE(0);
  pdl_begin(P);
  if constexpr (sizeof(T) == 4) {
    const Tile t = tile_of(P);
    const FeedDev<T> f = feed_of(P, t.member);
    // m0 = first input tile, layer = input tiles in the group, n0 = unit tile
    __shared__ MemberDev<float> sM;
    if (threadIdx.x < sizeof(MemberDev<float>) / 4)
      reinterpret_cast<int32_t*>(&sM)[threadIdx.x] =
          reinterpret_cast<const int32_t*>(mem_of(P, t.member))[threadIdx.x];
    __syncthreads();
    if (f.take != 0 && !halted(P)) m1t_bwd_tile(smem_raw, sM, f, t.m0, t.layer, t.n0, P.stages, P.gsize);
  } else {
    __trap();
  }
  kernel_end(P, true);
}

template <typename T>
__global__ void __launch_bounds__(NT, 1) k_mlp1_fwd(const __grid_constant__ PhaseArgs<T> P) {
  extern __shared__ __align__(16) char smem_raw[];
  if (threadIdx.x == 0)
    pk_trace_slots = P.trace ? P.trace + (size_t)blockIdx.x * kTraceSlots : nullptr;
  PK_TRACE(0);
  pdl_begin(P);
  if (P.prefetch) prefetch_params(P);
  const Tile t = tile_of(P);
  const FeedDev<T> f = feed_of(P, t.member);
  if (f.take != 0 && !halted(P)) m1_fwd_tile<T>(smem_raw, P.mems[t.member], f, t.m0);
  kernel_end(P, true);
}

template <typename T>
__global__ void __launch_bounds__(NT, 1) k_mlp1_bwd(const __grid_constant__ PhaseArgs<T> P) {
  extern __shared__ __align__(16) char smem_raw[];
  if (threadIdx.x == 0)
    pk_trace_slots = P.trace ? P.trace + (size_t)blockIdx.x * kTraceSlots : nullptr;
  PK_TRACE(0);
  pdl_begin(P);
  const Tile t = tile_of(P);
  const FeedDev<T> f = feed_of(P, t.member);
  if (f.take != 0 && !halted(P)) {
    const MemberDev<T>& M = P.mems[t.member];
    m1_bwd_tile<T>(smem_raw, M, f, t.m0, (M.dims[1] + M1_BC - 1) / M1_BC);
  }
  kernel_end(P, true);
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
