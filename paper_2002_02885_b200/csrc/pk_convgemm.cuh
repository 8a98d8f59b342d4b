// pk_convgemm.cuh — grouped implicit-GEMM convolution on tcgen05 (bf16 → fp32 TMEM).
//
// The dense conv and linear layers of the conv pack path
// are three GEMM shapes over NHWC bf16 activations:
//   FPROP  Y[m = (n,p,q), co]  = Σ_k  X[n, p·st−pad+r, q·st−pad+s, ci] · W[co, k]
//          k = (r, s, ci), ci fastest; A gathered (im2col) by cp.async, B = W by TMA.
//   DGRAD  dX[m = (n,h,w), ci] = Σ_k dY[n, (h+pad−r)/st, (w+pad−s)/st, co] · Wt[ci, k]
//          k = (r, s, co); taps whose quotient is not exact are zero; B = Wt by TMA
//          (a transposed bf16 copy the optimizer writes next to W).
//   WGRAD  dW[co, n = (r,s,ci)] = Σ_pix dY[pix, co] · X[im2col(pix), n]
//          both operands MN-major (pixel rows), gathered by cp.async; the pixel
//          reduction may be split (fixed split boundaries; the optimizer sums the
//          split partials in split order, so the result never depends on timing).
// One launch covers up to kMaxProblems problems — the K members of a pack at
// one layer (ragged rows / shapes allowed).  A CTA owns one 128 x NT output
// tile of one problem; problems never share a tile, and every output element's
// reduction order (64-deep K blocks in order, UMMA K=16 steps in order) is fixed
// by the problem's own shape, so a member's result is independent of the pack
// it trains in (packed == standalone bit for bit).
//
// Warp roles (192 threads): warps 0-3 gather operands with cp.async (16-B
// chunks, zero fill for padding / out-of-image taps) and then run the
// epilogue (TMEM lane quarter = warp); warp 4 owns TMEM and one lane issues the
// tcgen05.mma chain; warp 5 lane 0 issues the TMA loads of the weight operand.
// Stages ring through full/empty mbarriers; the producers' arrival on a
// stage lags one stage behind its issue (cp.async.wait_group 1 → proxy fence →
// arrive), so copies of consecutive stages overlap.
#pragma once
#include "pk_tc.cuh"

namespace cg {

enum Mode { FPROP = 0, DGRAD = 1, WGRAD = 2 };
constexpr int BM = 128, BK = 64;
constexpr int kMaxProblems = 16;
constexpr int kThreads = 192;

struct Problem {
  const __nv_bfloat16* src;   // gather source: X (FPROP/WGRAD) or dY (DGRAD)
  const __nv_bfloat16* src2;  // WGRAD: dY (the A operand)
  void* dst;                  // bf16 Y / dX, fp32 Y (out_f32), or fp32 dW partials
  const long long* idx;       // FPROP/WGRAD: image n of the batch is source image idx[n]
  const float* bias;          // FPROP epilogue: + bias[n] (NULL = none)
  int* flag;                  // WGRAD: set to 1 when a written gradient is non-finite
  int M, N, K;                // GEMM extents (K = true reduction extent, unpadded)
  int kper;                   // WGRAD: pixels per split (multiple of 64); else 0
  int tiles_m, tiles_n, splits, tile0;
  int pair0;                  // clustered launches: first M-tile pair of this problem
  int pw;                     // halo launches (k_conv_gemm_halo): padded row width W + 2 of the
                              //   output-pixel index space (0 = plain m = (n, y, x) rows)
  int tpi;                    // halo: M tiles per image
  int hrows;                  // halo: input rows per halo buffer
  int par;                    // stride-2 DGRAD parity class a·2 + b of the dX pixels
                              //   (2i + a, 2j + b) this problem computes, -1 = none; the
                              //   GEMM's pixel space is the (i, j) sub-grid OH x OW
  int DH, DW;                 // parity: dX plane dims
  int ntap;                   // parity (a_mode 5): the class's taps: global tap index r·S + s
  int tapk[4], tdr[4], tds[4];//   and the dY offsets (dr, ds) of (i, j) it reads
  int brow0;                  // FPROP/DGRAD: first row of this problem's B in its map
  const uint8_t* wbase;       // FPROP/DGRAD: the B (weight) matrix, row pitch wpitch bytes
  int wpitch;                 //   (L2 prefetch of a tile's panel before the PDL wait; 0 = off)
  int SH, SW, SC, sld;        // source tensor: spatial dims, channels, pixel stride
  int OH, OW;                 // spatial dims of the GEMM's pixel space
  int R, S, stride, pad;
  int dld;                    // dst row stride (elements)
  int ald;                    // WGRAD: dY pixel stride
  int nseg;                   // FPROP: columns per dst segment (concat-N), 0 = one
  int accumulate;             // DGRAD: dst += result
  int act;                    // FPROP epilogue activation after bias: 0 none, 1 relu, 2 relu6
  int out_f32;                // FPROP: dst is fp32
  int a_mode;                 // activation operand: 0 cp.async gather, 1 TMA 2-D tile,
                              //   2 TMA im2col (C % 64 == 0, SW128), 3 TMA im2col of a
                              //   16-channel input (one tap per 16-deep K chunk, SW32;
                              //   weights then also SW32) (FPROP/DGRAD: A; WGRAD: A=dY
                              //   is TMA 2-D whenever b_mode != 0)
  int b_mode;                 // WGRAD X operand: 0 gather, 1 TMA 2-D tile, 2 TMA im2col,
                              //   3 TMA im2col of a 16-channel input (SW32)
  int swap;                   // WGRAD (TMA, co <= 64): GEMM M = (r,s,c), N = co, so the
                              //   M = 128 MMA is not half empty; dst written transposed
  int wseg;                   // WGRAD, swapped: members concatenated along N (the shared-
                              //   input first layer), wseg = 64 columns each; dY atoms come
                              //   from a 3-D map {co, pixel, member}, member seg's partials
                              //   at dst + seg * dseg
  long long dseg;             // elements between dst segments
  long long split_stride;     // WGRAD: elements between split partials
};

struct Launch {
  CUtensorMap tm[kMaxProblems];   // FPROP/DGRAD: weights; WGRAD: X (b_mode != 0)
  CUtensorMap tmA[kMaxProblems];  // activation operand map (a_mode / WGRAD dY)
  Problem p[kMaxProblems];
  int nprob;
  int ntile;   // N tile: multiple of 16 in [16, 256] (multiple of 64 for WGRAD)
  int stages;  // pipeline depth
  int total_tiles;
  int persistent;  // every problem TMA-fed: k_conv_gemm_p, grid < total_tiles
  int grid;
  int cluster;     // 2: k_conv_gemm_pc — CTA pairs own adjacent M tiles and multicast
                   //    the shared B operand (weights), each loading one half
  int pair_mma;    // with cluster 2: k_conv_gemm_p2 — one M=256 tcgen05.mma.cta_group::2
                   //    per k-step over the pair (each CTA holds its A rows + half of B)
  int total_pairs;
  int halo;        // k_conv_gemm_halo (3x3 stride-1 FPROP / DGRAD, C % 64 == 0);
                   // 2: the weights-resident form k_conv_gemm_halo_res (C == 64, N <= 64)
  int abytes;      // halo: bytes of one halo buffer (1024-aligned)
};

__host__ __device__ inline uint32_t stage_bytes(int ntile) { return 16384u + (uint32_t)ntile * 128u; }
__host__ inline size_t smem_bytes(int ntile, int stages) {
  return 1024 + (size_t)stages * stage_bytes(ntile) + 8 * (2 * stages + 4) + 16;
}

// Issue the TMA loads of one 64-deep k-block (reduction offset kk) of tile
// (tm, tn) of problem pi into one pipeline stage, completing on `bar`.
//   FPROP/DGRAD: B = weights (2-D), and A when tma_all (2-D tile or im2col);
//   WGRAD (tma_all only): A = dY (2-D, two 64-wide M atoms), B = X (2-D or
//   im2col, NT/64 N atoms).
template <int MODE>
__device__ __forceinline__ void tma_kblock(const Launch& L, int pi, int tm, int tn, int kk,
                                           bool tma_all, uint8_t* stage, uint64_t* bar, int NT) {
  const Problem& P = L.p[pi];
  const int ohw = P.OH * P.OW;
  if (MODE == WGRAD) {
    umma::mbar_arrive_expect_tx(bar, 16384u + (uint32_t)NT * 128u);
    uint8_t* b_s = stage + 16384;
    const int img = kk / ohw, rem = kk - img * ohw;
    const int py = rem / P.OW, px = rem - py * P.OW;
    // one 64-wide atom of the X operand: columns n .. n+63 of (r, s, c)
    auto x_atom = [&](uint8_t* dst, int n) {
      if (P.b_mode == 3) {  // four 16-channel taps, 2 KB SW32 boxes
        for (int i = 0; i < 4; ++i) {
          const int tap = (n >> 4) + i, fr = tap / P.S, fs = tap - fr * P.S;
          tc::tma_im2col_4d(dst + i * 2048, &L.tm[pi], 0, px * P.stride - P.pad,
                            py * P.stride - P.pad, img, (uint16_t)fs, (uint16_t)fr, bar);
        }
      } else if (P.b_mode == 1) {
        tc::tma_load_2d(dst, &L.tm[pi], n, kk, bar);
      } else {
        const int tap = n / P.SC, c0 = n - tap * P.SC;
        const int fr = tap / P.S, fs = tap - fr * P.S;
        tc::tma_im2col_4d(dst, &L.tm[pi], c0, px * P.stride - P.pad, py * P.stride - P.pad, img,
                          (uint16_t)fs, (uint16_t)fr, bar);
      }
    };
    if (P.swap) {  // A = X (M = (r,s,c)), B = dY (N = co)
      x_atom(stage, tm * BM);
      x_atom(stage + 8192, tm * BM + 64);
      for (int j = 0; j < NT / 64; ++j) {
        if (P.wseg)
          tc::tma_load_3d(b_s + j * 8192, &L.tmA[pi], 0, kk, (tn * NT) / 64 + j, bar);
        else
          tc::tma_load_2d(b_s + j * 8192, &L.tmA[pi], tn * NT + j * 64, kk, bar);
      }
    } else {       // A = dY (M = co), B = X (N = (r,s,c))
      tc::tma_load_2d(stage, &L.tmA[pi], tm * BM, kk, bar);
      tc::tma_load_2d(stage + 8192, &L.tmA[pi], tm * BM + 64, kk, bar);
      for (int j = 0; j < NT / 64; ++j) x_atom(b_s + j * 8192, tn * NT + j * 64);
    }
    return;
  }
  umma::mbar_arrive_expect_tx(bar, (uint32_t)NT * 128u + (tma_all ? 16384u : 0u));
  const int m0 = tm * BM;
  if (P.a_mode == 6) {  // 32-channel plane: taps 2kb, 2kb+1, one SW64 slab each (DGRAD)
    const int img = m0 / ohw, rem = m0 - img * ohw;
    const int py = rem / P.OW, px = rem - py * P.OW;
    const int kb = kk / BK, ntaps = P.R * P.S;
    for (int u = 0; u < 2; ++u) {
      const int tb = 2 * kb + u;           // B: past the last tap these are zero columns
      const int tap = min(tb, ntaps - 1);  // A: a real (finite) tap that meets zero B rows
      const int fr = tap / P.S, fs = tap - fr * P.S;
      tc::tma_im2col_4d(stage + u * 8192, &L.tmA[pi], 0, px + P.pad - (P.S - 1),
                        py + P.pad - (P.R - 1), img, (uint16_t)(P.S - 1 - fs),
                        (uint16_t)(P.R - 1 - fr), bar);
      tc::tma_load_2d(stage + 16384 + u * NT * 64, &L.tm[pi], tb * 32, P.brow0 + tn * NT, bar);
    }
    return;
  }
  if (P.a_mode == 5) {  // stride-2 DGRAD parity class: tap t of the class, dY at (i+dr, j+ds)
    const int img = m0 / ohw, rem = m0 - img * ohw;
    const int py = rem / P.OW, px = rem - py * P.OW;
    const int t = kk / P.SC, c0 = kk - t * P.SC;
    tc::tma_im2col_4d(stage, &L.tmA[pi], c0, px, py, img, (uint16_t)P.tds[t], (uint16_t)P.tdr[t],
                      bar);
    tc::tma_load_2d(stage + 16384, &L.tm[pi], P.tapk[t] * P.SC + c0, P.brow0 + tn * NT, bar);
    return;
  }
  if (P.a_mode == 3) {  // four taps of a 16-channel input: A and B in 16-deep SW32 slabs
    const int img = m0 / ohw, rem = m0 - img * ohw;
    const int py = rem / P.OW, px = rem - py * P.OW;
    for (int i = 0; i < 4; ++i) {
      const int tap = (kk >> 4) + i, fr = tap / P.S, fs = tap - fr * P.S;
      tc::tma_im2col_4d(stage + i * 4096, &L.tmA[pi], 0, px * P.stride - P.pad,
                        py * P.stride - P.pad, img, (uint16_t)fs, (uint16_t)fr, bar);
      tc::tma_load_2d(stage + 16384 + i * NT * 32, &L.tm[pi], kk + 16 * i, P.brow0 + tn * NT,
                      bar);
    }
    return;
  }
  if (P.a_mode == 1) {
    tc::tma_load_2d(stage, &L.tmA[pi], kk, m0, bar);
  } else if (P.a_mode == 2) {
    const int img = m0 / ohw, rem = m0 - img * ohw;
    const int py = rem / P.OW, px = rem - py * P.OW;
    const int tap = kk / P.SC, c0 = kk - tap * P.SC;
    const int fr = tap / P.S, fs = tap - fr * P.S;
    if (MODE == FPROP)
      tc::tma_im2col_4d(stage, &L.tmA[pi], c0, px * P.stride - P.pad, py * P.stride - P.pad, img,
                        (uint16_t)fs, (uint16_t)fr, bar);
    else  // stride-1 data gradient: dY window of dX pixel (y, x), taps reversed
      tc::tma_im2col_4d(stage, &L.tmA[pi], c0, px + P.pad - (P.S - 1), py + P.pad - (P.R - 1),
                        img, (uint16_t)(P.S - 1 - fs), (uint16_t)(P.R - 1 - fr), bar);
  }
  tc::tma_load_2d(stage + 16384, &L.tm[pi], kk, P.brow0 + tn * NT, bar);
}

// 4 UMMA K-steps (K = 16 each) of one stage into the accumulator at tmem_d.
// sw32a / sw32b: that operand is in 32-byte-swizzled slabs (16-channel input).
template <int MODE>
__device__ __forceinline__ void mma_kblock(uint32_t tmem_d, uint32_t a_s, uint32_t idesc,
                                           bool first, bool sw32a = false, bool sw32b = false,
                                           int NT = 0) {
  const uint32_t b_s = a_s + 16384;
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    uint64_t ad, bd;
    if (MODE == WGRAD) {  // MN-major operands
      ad = sw32a ? tc::sdesc_sw32(a_s + ks * 512, 2048, 256)
                 : tc::sdesc_sw128(a_s + ks * 2048, 8192, 1024);
      bd = sw32b ? tc::sdesc_sw32(b_s + ks * 512, 2048, 256)
                 : tc::sdesc_sw128(b_s + ks * 2048, 8192, 1024);
    } else {              // K-major operands
      ad = sw32a ? tc::sdesc_sw32(a_s + ks * 4096, 16, 256)
                 : tc::sdesc_sw128(a_s + ks * 32, 16, 1024);
      bd = sw32b ? tc::sdesc_sw32(b_s + ks * NT * 32, 16, 256)
                 : tc::sdesc_sw128(b_s + ks * 32, 16, 1024);
    }
    tc::mma_bf16(tmem_d, ad, bd, idesc, (!first || ks) ? 1u : 0u);
  }
}

// 4 UMMA K-steps of a 32-channel (a_mode 6) stage: two SW64 slabs of 32 K each
__device__ __forceinline__ void mma_kblock_sw64(uint32_t tmem_d, uint32_t a_s, uint32_t idesc,
                                                bool first, int NT) {
  const uint32_t b_s = a_s + 16384;
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const uint32_t u = ks >> 1, h = (ks & 1) * 32;
    tc::mma_bf16(tmem_d, tc::sdesc_sw64(a_s + u * 8192 + h, 16, 512),
                 tc::sdesc_sw64(b_s + u * NT * 64 + h, 16, 512), idesc,
                 (!first || ks) ? 1u : 0u);
  }
}

// which operands of problem P sit in SW32 slabs
__device__ __forceinline__ void sw32_flags(const Problem& P, bool wgrad, bool& a, bool& b) {
  if (wgrad) {
    const bool x = P.b_mode == 3;
    a = P.swap ? x : false;
    b = P.swap ? false : x;
  } else {
    a = b = P.a_mode == 3;
  }
}

struct TileInfo {
  int pi, split, tm, tn, k0, nkb;
};
__device__ __forceinline__ TileInfo decode_tile(const Launch& L, int t, bool wgrad) {
  TileInfo T;
  int pi = 0;
  while (pi + 1 < L.nprob && t >= L.p[pi + 1].tile0) ++pi;
  const Problem& P = L.p[pi];
  int lt = t - P.tile0;
  const int per_split = P.tiles_m * P.tiles_n;
  T.pi = pi;
  T.split = lt / per_split;
  lt -= T.split * per_split;
  T.tm = lt % P.tiles_m;
  T.tn = lt / P.tiles_m;
  int k0 = 0, kend = P.K;
  if (wgrad) {
    k0 = T.split * P.kper;
    kend = min(P.K, k0 + P.kper);
  }
  T.k0 = k0;
  T.nkb = (kend - k0 + BK - 1) / BK;
  return T;
}

// The weights do not depend on the previous kernel of the step (they were written by
// the previous step's optimizer / transpose, in an earlier graph launch), so the TMA
// producer pulls its first tile's weight panel into L2 before griddepcontrol.wait:
// the first k-blocks' B loads then hit L2 while A waits on the predecessor.
template <int MODE>
__device__ __forceinline__ void prefetch_b_panel(const Launch& L, int t, int NT) {
  if (MODE == WGRAD || t >= L.total_tiles) return;
  const TileInfo ti = decode_tile(L, t, false);
  const Problem& P = L.p[ti.pi];
  if (!P.wbase || P.wpitch <= 0) return;
  const int rows = min(NT, P.N - ti.tn * NT);
  if (rows <= 0) return;
  const uint8_t* a = P.wbase + ((long long)P.brow0 + (long long)ti.tn * NT) * P.wpitch;
  // short-K GEMMs only (<= four 64-deep k-blocks: the 1x1 convs of the small nets, whose
  // launches are latency-bound): the whole panel in one contiguous bulk prefetch. Longer
  // rows measured slower (config3 +0.05-0.12 ms: per-row prefetches delay the producer)
  if (P.wpitch <= 4 * BK * 2)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a),
                 "r"((uint32_t)(rows * P.wpitch)) : "memory");
}

// TMEM accumulator (columns [tcol, tcol + NT) of this CTA's allocation) of one
// output tile → global: bias / activation / fp32 / concat-N / accumulate per
// the problem, non-finite flag for WGRAD.  Warps 0-3, lane quarter = warp.
template <int MODE>
__device__ __forceinline__ void epilogue(const Problem& P, uint32_t tmem, int warp, int lane,
                                         int tm, int tn, int split, int nkb, int NT) {
  const int row = warp * 32 + lane;
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  int m = tm * BM + row;     // the output row written (dst row index)
  bool mvalid = m < P.M;
  if (P.par >= 0) {  // stride-2 DGRAD parity class: (n, i, j) → dX pixel (2i + a, 2j + b)
    const int ohw = P.OH * P.OW, n = m / ohw, rem = m - n * ohw;
    const int i = rem / P.OW, j = rem - i * P.OW;
    m = (n * P.DH + 2 * i + (P.par >> 1)) * P.DW + 2 * j + (P.par & 1);
  }
  if (P.pw) {  // halo tiles: rows index the padded (W + 2)-wide pixels of one image
    const int img = tm / P.tpi, o = (tm - img * P.tpi) * BM + row;
    const int y = o / P.pw, x = o - y * P.pw;
    mvalid = y < P.OH && x < P.OW;  // junk columns / rows past the image are dropped
    m = mvalid ? (img * P.OH + y) * P.OW + x : 0;
  }
  // one 16-column chunk of the accumulator row → global
  auto chunk = [&](int c0, float (&v)[16]) {    const int n0 = tn * NT + c0;
    if (!mvalid || n0 >= P.N) return;
    if (MODE == FPROP && (P.bias || P.act)) {
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        float x = v[e];
        if (P.bias) x += (n0 + e < P.N) ? __ldg(P.bias + n0 + e) : 0.f;
        if (P.act == 1) x = fmaxf(x, 0.f);
        else if (P.act == 2) x = fminf(fmaxf(x, 0.f), 6.f);
        v[e] = x;
      }
    }
    if (MODE == WGRAD && P.flag) {
      bool bad = false;
#pragma unroll
      for (int e = 0; e < 16; ++e) bad |= (n0 + e < P.N) && !isfinite(v[e]);
      if (bad) *P.flag = 1;
    }
    if (MODE == FPROP && P.out_f32) {
      float* d = static_cast<float*>(P.dst) + (long long)m * P.dld + n0;
      if (n0 + 16 <= P.N && (P.dld & 3) == 0) {
#pragma unroll
        for (int e = 0; e < 16; e += 4)
          *reinterpret_cast<float4*>(d + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
      } else {
        for (int e = 0; e < 16 && n0 + e < P.N; ++e) d[e] = v[e];
      }
    } else if (MODE == WGRAD && P.swap) {
      // accumulator row m = (r,s,c) column of dW, columns = co rows of dW
      float* d = static_cast<float*>(P.dst) + (long long)split * P.split_stride + m;
      if (P.wseg) {  // 16 | wseg: the 16 columns belong to one member
        const int seg = n0 / P.wseg;
        d += seg * P.dseg - (long long)seg * P.wseg * P.dld;
      }
      for (int e = 0; e < 16 && n0 + e < P.N; ++e) d[(long long)(n0 + e) * P.dld] = v[e];
    } else if (MODE == WGRAD) {
      float* d = static_cast<float*>(P.dst) + (long long)split * P.split_stride +
                 (long long)m * P.dld + n0;
      if (n0 + 16 <= P.N) {
#pragma unroll
        for (int e = 0; e < 16; e += 4)
          *reinterpret_cast<float4*>(d + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
      } else {
        for (int e = 0; e < 16 && n0 + e < P.N; ++e) d[e] = v[e];
      }
    } else {
      int seg = 0, nn = n0;
      if (P.nseg > 0) {
        seg = n0 / P.nseg;
        nn = n0 - seg * P.nseg;
      }
      __nv_bfloat16* d = static_cast<__nv_bfloat16*>(P.dst) + (long long)seg * P.dseg +
                         (long long)m * P.dld + nn;
      const bool vec = n0 + 16 <= P.N && (P.nseg == 0 || nn + 16 <= P.nseg);
      if (vec) {
        if (P.accumulate) {
          const uint4 o0 = reinterpret_cast<const uint4*>(d)[0];
          const uint4 o1 = reinterpret_cast<const uint4*>(d)[1];
          const __nv_bfloat16* ob0 = reinterpret_cast<const __nv_bfloat16*>(&o0);
          const __nv_bfloat16* ob1 = reinterpret_cast<const __nv_bfloat16*>(&o1);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            v[e] += __bfloat162float(ob0[e]);
            v[e + 8] += __bfloat162float(ob1[e]);
          }
        }
        uint4 w0, w1;
        w0.x = tc::pack_bf16(v[0], v[1]);
        w0.y = tc::pack_bf16(v[2], v[3]);
        w0.z = tc::pack_bf16(v[4], v[5]);
        w0.w = tc::pack_bf16(v[6], v[7]);
        w1.x = tc::pack_bf16(v[8], v[9]);
        w1.y = tc::pack_bf16(v[10], v[11]);
        w1.z = tc::pack_bf16(v[12], v[13]);
        w1.w = tc::pack_bf16(v[14], v[15]);
        reinterpret_cast<uint4*>(d)[0] = w0;
        reinterpret_cast<uint4*>(d)[1] = w1;
      } else {
        for (int e = 0; e < 16 && n0 + e < P.N; ++e) {
          int sg = seg, cn = nn + e;
          if (P.nseg > 0 && cn >= P.nseg) {
            sg += cn / P.nseg;
            cn -= (cn / P.nseg) * P.nseg;
          }
          __nv_bfloat16* de = static_cast<__nv_bfloat16*>(P.dst) + (long long)sg * P.dseg +
                              (long long)m * P.dld + cn;
          float x = v[e];
          if (P.accumulate) x += __bfloat162float(*de);
          *de = __float2bfloat16_rn(x);
        }
      }
    }
    };
  // TMEM → registers 32 columns per tcgen05.ld (one wait per 32 columns)
  for (int c1 = 0; c1 < NT; c1 += 32) {
    float w[2][16];
    const bool two = c1 + 32 <= NT;
    if (nkb > 0) {
      if (two) tc::tmem_ld32(trow + c1, w[0], w[1]);
      else tc::tmem_ld16(trow + c1, w[0]);
    } else {
#pragma unroll
      for (int e = 0; e < 16; ++e) w[0][e] = w[1][e] = 0.f;
    }
    chunk(c1, w[0]);
    if (two) chunk(c1 + 16, w[1]);
  }
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 2)
k_conv_gemm(const __grid_constant__ Launch L) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int NT = L.ntile, ST = L.stages;
  const uint32_t SB = stage_bytes(NT);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * SB);
  uint64_t* empty = full + ST;
  uint64_t* done = empty + ST;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- tile → (problem, split, m tile, n tile) ----
  int pi = 0;
  const int t = blockIdx.x;
  while (pi + 1 < L.nprob && t >= L.p[pi + 1].tile0) ++pi;
  const Problem& P = L.p[pi];
  int lt = t - P.tile0;
  const int per_split = P.tiles_m * P.tiles_n;
  const int split = lt / per_split;
  lt -= split * per_split;
  const int tm = lt % P.tiles_m, tn = lt / P.tiles_m;
  int k0 = 0, kend = P.K;
  if (MODE == WGRAD) {
    k0 = split * P.kper;
    kend = min(P.K, k0 + P.kper);
  }
  const int nkb = (kend - k0 + BK - 1) / BK;
  // which operands the TMA warp loads: all (tma_all) or only the FPROP/DGRAD weights
  const bool tma_all = MODE == WGRAD ? P.b_mode != 0 : P.a_mode != 0;
  const bool kTma = MODE != WGRAD || tma_all;

  if (tid == 160) {
    for (int s = 0; s < ST; ++s) {
      umma::mbar_init(&full[s], tma_all ? 1 : 128 + (kTma ? 1 : 0));
      umma::mbar_init(&empty[s], 1);
    }
    umma::mbar_init(done, 1);
    umma::mbar_fence_init();
    if (kTma) tc::tma_prefetch(&L.tm[pi]);
    if (tma_all) tc::tma_prefetch(&L.tmA[pi]);
  }
  const uint32_t tcols = umma::tmem_cols_pow2((uint32_t)NT);
  if (warp == 4) umma::tmem_alloc(tmem_slot, tcols);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 160) prefetch_b_panel<MODE>(L, blockIdx.x, L.ntile);

  tc::pdl_gate();

  if (warp < 4) {
    // =========================== producers ===========================
    const uint32_t sbase = tc::smem_u32(smem);
    if (tma_all) {
      // operands arrive by TMA (warp 5): these warps only run the epilogue
    } else if (MODE != WGRAD) {
      const int j = tid & 7, r0 = tid >> 3;
      int rimg[8], ry[8], rx[8];
      const int ohw = P.OH * P.OW;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int m = tm * BM + r0 + 16 * i;
        if (m < P.M) {
          const int n = m / ohw, rem = m - n * ohw, y = rem / P.OW, x = rem - y * P.OW;
          rimg[i] = (MODE == FPROP && P.idx ? (int)P.idx[n] : n) * P.SH * P.SW;
          if (MODE == FPROP) {
            ry[i] = y * P.stride - P.pad;
            rx[i] = x * P.stride - P.pad;
          } else {
            ry[i] = y + P.pad;
            rx[i] = x + P.pad;
          }
        } else {
          rimg[i] = -1;
          ry[i] = rx[i] = 0;
        }
      }
      const int sh = P.stride - 1;  // stride in {1, 2}
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % ST;
        if (kb >= ST) umma::mbar_wait(&empty[s], ((kb / ST) + 1) & 1);
        const uint32_t a_s = sbase + s * SB;
        const int k = k0 + kb * BK + 8 * j;
        const int tap = k / P.SC, c = k - tap * P.SC;
        const int r = tap / P.S, sx = tap - r * P.S;
        const bool kok = k < kend;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          int iy, ix;
          bool ok = kok && rimg[i] >= 0;
          if (MODE == FPROP) {
            iy = ry[i] + r;
            ix = rx[i] + sx;
          } else {
            const int ny = ry[i] - r, nx = rx[i] - sx;
            ok = ok && ny >= 0 && nx >= 0 && ((ny | nx) & sh) == 0;
            iy = ny >> sh;
            ix = nx >> sh;
          }
          ok = ok && (unsigned)iy < (unsigned)P.SH && (unsigned)ix < (unsigned)P.SW;
          const __nv_bfloat16* g =
              ok ? P.src + ((long long)(rimg[i] + iy * P.SW + ix) * P.sld + c) : P.src;
          tc::cp16(a_s + tc::kmaj_sw128(r0 + 16 * i, j), g, ok);
        }
        tc::cp_commit();
        if (kb >= 1) {
          tc::cp_wait<1>();
          umma::fence_async_smem();
          tc::mbar_arrive(&full[(kb - 1) % ST]);
        }
      }
    } else {
      // A: dY [64 pixel rows][128 co], MN-major
      const int acj = tid & 15, arr = tid >> 4;
      const int co = tm * BM + acj * 8;
      const bool co_ok = co < P.M;
      // B: X im2col [64 pixel rows][NT cols], MN-major
      const int cpr = NT >> 3, rpp = 128 / cpr, passes = BK / rpp;
      const int bcj = tid % cpr, brr = tid / cpr;
      const int col = tn * NT + bcj * 8;
      const int tap = col / P.SC, cc = col - tap * P.SC;
      const int fr = tap / P.S, fs = tap - fr * P.S;
      const bool col_ok = col < P.N;
      const int ohw = P.OH * P.OW;
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % ST;
        if (kb >= ST) umma::mbar_wait(&empty[s], ((kb / ST) + 1) & 1);
        const uint32_t a_s = sbase + s * SB, b_s = a_s + 16384;
        const int kbase = k0 + kb * BK;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int row = arr + 8 * i, pix = kbase + row;
          const bool ok = co_ok && pix < kend;
          const __nv_bfloat16* g = ok ? P.src2 + ((long long)pix * P.ald + co) : P.src2;
          tc::cp16(a_s + tc::mnmaj_sw128(row, acj), g, ok);
        }
        for (int ps = 0; ps < passes; ++ps) {
          const int row = brr + ps * rpp, pix = kbase + row;
          bool ok = col_ok && pix < kend;
          long long off = 0;
          if (ok) {
            const int n = pix / ohw, rem = pix - n * ohw, y = rem / P.OW, x = rem - y * P.OW;
            const int iy = y * P.stride - P.pad + fr, ix = x * P.stride - P.pad + fs;
            ok = (unsigned)iy < (unsigned)P.SH && (unsigned)ix < (unsigned)P.SW;
            const long long img = P.idx ? P.idx[n] : n;
            off = ((img * P.SH + iy) * P.SW + ix) * P.sld + cc;
          }
          tc::cp16(b_s + tc::mnmaj_sw128(row, bcj), ok ? P.src + off : P.src, ok);
        }
        tc::cp_commit();
        if (kb >= 1) {
          tc::cp_wait<1>();
          umma::fence_async_smem();
          tc::mbar_arrive(&full[(kb - 1) % ST]);
        }
      }
    }
    if (nkb > 0 && !tma_all) {
      tc::cp_wait<0>();
      umma::fence_async_smem();
      tc::mbar_arrive(&full[(nkb - 1) % ST]);
    }

    // =========================== epilogue ===========================
    umma::mbar_wait(done, 0);
    umma::fence_after();
    epilogue<MODE>(P, tmem, warp, lane, tm, tn, split, nkb, NT);
  } else if (warp == 4) {
    // =========================== MMA issuer ===========================
    if (lane == 0) {
      constexpr bool mn = MODE == WGRAD;
      const uint32_t idesc = tc::idesc_bf16(BM, NT, mn, mn);
      const uint32_t sbase = tc::smem_u32(smem);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % ST;
        umma::mbar_wait(&full[s], (kb / ST) & 1);
        umma::fence_after();
        bool fa, fb;
        sw32_flags(P, MODE == WGRAD, fa, fb);
        if (MODE != WGRAD && P.a_mode == 6)
          mma_kblock_sw64(tmem, sbase + s * SB, idesc, kb == 0, NT);
        else
          mma_kblock<MODE>(tmem, sbase + s * SB, idesc, kb == 0, fa, fb, NT);
        umma::commit(&empty[s]);
      }
      umma::commit(done);
    }
    __syncwarp();
  } else if (kTma && warp == 5 && lane == 0) {
    // =========================== TMA ===========================
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % ST;
      if (kb >= ST) umma::mbar_wait(&empty[s], ((kb / ST) + 1) & 1);
      tma_kblock<MODE>(L, pi, tm, tn, k0 + kb * BK, tma_all, smem + s * SB, &full[s], NT);
    }
  }

  umma::fence_before();
  __syncthreads();
  if (warp == 4) {
    umma::fence_after();
    umma::tmem_dealloc(tmem, tcols);
  }
}

// ------------------------------------------------------------------------------
// Persistent variant, for launches whose operands all arrive by TMA.  A CTA
// walks tiles blockIdx.x, +gridDim.x, ...; the smem ring runs continuously
// across tiles (warp 5 keeps loading the next tile's k-blocks while the last
// ones are multiplied), and two TMEM accumulators (columns [0, NT) and
// [S, S+NT), S = half the power-of-two allocation) alternate between tiles so warps 0-3 drain tile i while warp 4
// issues tile i+1's MMAs.  Tile arithmetic is the one-tile kernel's, so
// results are identical bit for bit.
// ------------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(kThreads, 1) k_conv_gemm_p(const __grid_constant__ Launch L) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int NT = L.ntile, ST = L.stages;
  const uint32_t SB = stage_bytes(NT);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * SB);
  uint64_t* empty = full + ST;
  uint64_t* tfull = empty + ST;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr bool wg = MODE == WGRAD;
  if (tid == 160) {
    for (int s = 0; s < ST; ++s) {
      umma::mbar_init(&full[s], 1);
      umma::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      umma::mbar_init(&tfull[b], 1);
      umma::mbar_init(&tempty[b], 128);
    }
    umma::mbar_fence_init();
  }
  const uint32_t tcols = umma::tmem_cols_pow2((uint32_t)(2 * NT));
  if (warp == 4) umma::tmem_alloc(tmem_slot, tcols);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 160) prefetch_b_panel<MODE>(L, blockIdx.x, L.ntile);

  tc::pdl_gate();
  const uint32_t bstride = tcols / 2;  // accumulator buffer b at columns [b*bstride, +NT)
  const int T = L.total_tiles;

  if (warp == 5) {
    if (lane == 0) {  // ---- TMA producer ----
      int g = 0;
      for (int t = blockIdx.x; t < T; t += gridDim.x) {
        const TileInfo ti = decode_tile(L, t, wg);
        for (int kb = 0; kb < ti.nkb; ++kb, ++g) {
          const int s = g % ST;
          if (g >= ST) umma::mbar_wait(&empty[s], ((g / ST) + 1) & 1);
          tma_kblock<MODE>(L, ti.pi, ti.tm, ti.tn, ti.k0 + kb * BK, true, smem + s * SB, &full[s],
                           NT);
        }
      }
    }
  } else if (warp == 4) {
    if (lane == 0) {  // ---- MMA issuer ----
      const uint32_t idesc = tc::idesc_bf16(BM, NT, wg, wg);
      const uint32_t sbase = tc::smem_u32(smem);
      int g = 0, it = 0;
      for (int t = blockIdx.x; t < T; t += gridDim.x, ++it) {
        const TileInfo ti = decode_tile(L, t, wg);
        const int buf = it & 1;
        if (it >= 2) umma::mbar_wait(&tempty[buf], ((it >> 1) + 1) & 1);
        umma::fence_after();
        const uint32_t acc = tmem + (uint32_t)buf * bstride;
        for (int kb = 0; kb < ti.nkb; ++kb, ++g) {
          const int s = g % ST;
          umma::mbar_wait(&full[s], (g / ST) & 1);
          umma::fence_after();
          bool fa, fb;
          sw32_flags(L.p[ti.pi], wg, fa, fb);
          if (!wg && L.p[ti.pi].a_mode == 6)
            mma_kblock_sw64(acc, sbase + s * SB, idesc, kb == 0, NT);
          else
            mma_kblock<MODE>(acc, sbase + s * SB, idesc, kb == 0, fa, fb, NT);
          umma::commit(&empty[s]);
        }
        umma::commit(&tfull[buf]);
      }
    }
    __syncwarp();
  } else {  // ---- warps 0-3: epilogue ----
    int it = 0;
    for (int t = blockIdx.x; t < T; t += gridDim.x, ++it) {
      const TileInfo ti = decode_tile(L, t, wg);
      const int buf = it & 1;
      umma::mbar_wait(&tfull[buf], (it >> 1) & 1);
      umma::fence_after();
      epilogue<MODE>(L.p[ti.pi], tmem + (uint32_t)buf * bstride, warp, lane, ti.tm, ti.tn, ti.split,
                     ti.nkb, NT);
      umma::fence_before();
      tc::mbar_arrive(&tempty[buf]);
    }
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 4) {
    umma::fence_after();
    umma::tmem_dealloc(tmem, tcols);
  }
}

// ------------------------------------------------------------------------------
// Clustered persistent variant (FPROP / DGRAD with TMA-fed activations): the two
// CTAs of a cluster own M tiles 2i and 2i+1 of the same (problem, N tile) and
// share its B operand (the weights): each CTA's TMA thread loads its own A tile
// and HALF of the B box (NT/2 rows), multicast to both CTAs, so the L2 → SM
// traffic of B halves.  A stage is reusable only when both CTAs' MMAs have
// consumed it: every CTA commits its MMAs to the `empty` barrier of both CTAs
// (count 2).  The arithmetic per output element is the one-CTA kernel's, so
// results are identical bit for bit.
// ------------------------------------------------------------------------------
__device__ __forceinline__ TileInfo decode_pair(const Launch& L, int t2, int rank) {
  TileInfo T;
  int pi = 0;
  while (pi + 1 < L.nprob && t2 >= L.p[pi + 1].pair0) ++pi;
  const Problem& P = L.p[pi];
  const int tm2 = (P.tiles_m + 1) / 2;
  int lt = t2 - P.pair0;
  T.pi = pi;
  T.split = 0;
  T.tm = 2 * (lt % tm2) + rank;
  T.tn = lt / tm2;
  T.k0 = 0;
  T.nkb = (P.K + BK - 1) / BK;
  return T;
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1) k_conv_gemm_pc(const __grid_constant__ Launch L) {
  static_assert(MODE != WGRAD, "clustered variant: FPROP / DGRAD");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int NT = L.ntile, ST = L.stages;
  const uint32_t SB = stage_bytes(NT);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * SB);
  uint64_t* empty = full + ST;
  uint64_t* tfull = empty + ST;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rank = (int)tc::cluster_rank();
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  if (tid == 160) {
    for (int s = 0; s < ST; ++s) {
      umma::mbar_init(&full[s], 1);
      umma::mbar_init(&empty[s], 2);  // both CTAs' MMAs release a stage
    }
    for (int b = 0; b < 2; ++b) {
      umma::mbar_init(&tfull[b], 1);
      umma::mbar_init(&tempty[b], 128);
    }
    umma::mbar_fence_init();
  }
  const uint32_t tcols = umma::tmem_cols_pow2((uint32_t)(2 * NT));
  if (warp == 4) umma::tmem_alloc(tmem_slot, tcols);
  umma::fence_before();
  __syncthreads();
  umma::cluster_sync();  // the peer's barriers are initialised before any remote arrive
  umma::fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 160) prefetch_b_panel<MODE>(L, blockIdx.x, L.ntile);

  tc::pdl_gate();
  const uint32_t bstride = tcols / 2;
  const int T2 = L.total_pairs;
  const uint32_t half = (uint32_t)NT * 64u;  // bytes of half the B box (NT/2 rows x 128 B)

  if (warp == 5) {
    if (lane == 0) {  // ---- TMA producer: own A, half of the shared B (multicast) ----
      int g = 0;
      for (int t = cid; t < T2; t += ncl) {
        const TileInfo ti = decode_pair(L, t, rank);
        const Problem& P = L.p[ti.pi];
        const int ohw = P.OH * P.OW, m0 = ti.tm * BM;
        for (int kb = 0; kb < ti.nkb; ++kb, ++g) {
          const int s = g % ST;
          if (g >= ST) umma::mbar_wait(&empty[s], ((g / ST) + 1) & 1);
          uint8_t* stage = smem + s * SB;
          const int kk = kb * BK;
          umma::mbar_arrive_expect_tx(&full[s], 16384u + (uint32_t)NT * 128u);
          if (P.a_mode == 1) {
            tc::tma_load_2d(stage, &L.tmA[ti.pi], kk, m0, &full[s]);
          } else {
            const int img = m0 / ohw, rem = m0 - img * ohw;
            const int py = rem / P.OW, px = rem - py * P.OW;
            const int tap = kk / P.SC, c0 = kk - tap * P.SC;
            const int fr = tap / P.S, fs = tap - fr * P.S;
            if (MODE == FPROP)
              tc::tma_im2col_4d(stage, &L.tmA[ti.pi], c0, px * P.stride - P.pad,
                                py * P.stride - P.pad, img, (uint16_t)fs, (uint16_t)fr, &full[s]);
            else
              tc::tma_im2col_4d(stage, &L.tmA[ti.pi], c0, px + P.pad - (P.S - 1),
                                py + P.pad - (P.R - 1), img, (uint16_t)(P.S - 1 - fs),
                                (uint16_t)(P.R - 1 - fr), &full[s]);
          }
          tc::tma_load_2d_mc(stage + 16384 + rank * half, &L.tm[ti.pi], kk,
                             P.brow0 + ti.tn * NT + rank * (NT / 2), &full[s], (uint16_t)3);
        }
      }
    }
  } else if (warp == 4) {
    if (lane == 0) {  // ---- MMA issuer ----
      const uint32_t idesc = tc::idesc_bf16(BM, NT, false, false);
      const uint32_t sbase = tc::smem_u32(smem);
      int g = 0, it = 0;
      for (int t = cid; t < T2; t += ncl, ++it) {
        const TileInfo ti = decode_pair(L, t, rank);
        const int buf = it & 1;
        if (it >= 2) umma::mbar_wait(&tempty[buf], ((it >> 1) + 1) & 1);
        umma::fence_after();
        const uint32_t acc = tmem + (uint32_t)buf * bstride;
        for (int kb = 0; kb < ti.nkb; ++kb, ++g) {
          const int s = g % ST;
          umma::mbar_wait(&full[s], (g / ST) & 1);
          umma::fence_after();
          mma_kblock<MODE>(acc, sbase + s * SB, idesc, kb == 0, false, false, NT);
          tc::commit_mc(&empty[s], (uint16_t)3);
        }
        umma::commit(&tfull[buf]);
      }
    }
    __syncwarp();
  } else {  // ---- warps 0-3: epilogue ----
    int it = 0;
    for (int t = cid; t < T2; t += ncl, ++it) {
      const TileInfo ti = decode_pair(L, t, rank);
      const int buf = it & 1;
      umma::mbar_wait(&tfull[buf], (it >> 1) & 1);
      umma::fence_after();
      epilogue<MODE>(L.p[ti.pi], tmem + (uint32_t)buf * bstride, warp, lane, ti.tm, ti.tn, 0,
                     ti.nkb, NT);
      umma::fence_before();
      tc::mbar_arrive(&tempty[buf]);
    }
  }
  umma::fence_before();
  __syncthreads();
  umma::cluster_sync();  // no CTA leaves while its peer may still arrive on its barriers
  if (warp == 4) {
    umma::fence_after();
    umma::tmem_dealloc(tmem, tcols);
  }
}

// ------------------------------------------------------------------------------
// CTA-pair MMA variant (FPROP / DGRAD, TMA-fed activations).  The two CTAs of a
// cluster compute M tiles 2i, 2i+1 with ONE tcgen05.mma.cta_group::2 (M = 256)
// per K step, issued by the leader (rank 0): each CTA's smem holds its own 128 A
// rows and HALF of the B tile (NT/2 rows), so a stage costs 16 KB + NT·64 B per
// CTA instead of 16 KB + NT·128 B — deeper pipelines in the same shared memory.
// Both CTAs' TMA loads complete on the leader's `full` barrier; the leader's
// commits arrive on both CTAs' `empty` / `tfull` barriers (multicast); both
// epilogues release a TMEM buffer on the leader's `tempty` (8 warp arrivals).
// Each CTA's TMEM holds its 128 rows x NT columns: the epilogue is unchanged, and
// every output element's K order is the one-CTA kernel's.
// ------------------------------------------------------------------------------
__host__ __device__ inline uint32_t stage_bytes_pair(int ntile) {
  return 16384u + (uint32_t)ntile * 64u;
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1) k_conv_gemm_p2(const __grid_constant__ Launch L) {
  static_assert(MODE != WGRAD, "CTA-pair variant: FPROP / DGRAD");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int NT = L.ntile, ST = L.stages;
  const uint32_t SB = stage_bytes_pair(NT);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * SB);
  uint64_t* empty = full + ST;
  uint64_t* tfull = empty + ST;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rank = (int)tc::cluster_rank();
  const bool leader = rank == 0;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  if (tid == 160) {
    for (int s = 0; s < ST; ++s) {
      umma::mbar_init(&full[s], 1);   // leader: its producer's arrive + both CTAs' bytes
      umma::mbar_init(&empty[s], 1);  // the leader's MMA commit (multicast)
    }
    for (int b = 0; b < 2; ++b) {
      umma::mbar_init(&tfull[b], 1);
      umma::mbar_init(&tempty[b], 8);  // leader: 4 epilogue warps of each CTA
    }
    umma::mbar_fence_init();
  }
  const uint32_t tcols = umma::tmem_cols_pow2((uint32_t)(2 * NT));
  if (warp == 4) tc::tmem_alloc_pair(tmem_slot, tcols);
  umma::fence_before();
  __syncthreads();
  umma::cluster_sync();
  umma::fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 160) prefetch_b_panel<MODE>(L, blockIdx.x, L.ntile);

  tc::pdl_gate();
  const uint32_t bstride = tcols / 2;
  const int T2 = L.total_pairs;
  const uint32_t half = (uint32_t)NT * 64u;

  if (warp == 5) {
    if (lane == 0) {  // ---- TMA producer (both CTAs) ----
      int g = 0;
      for (int t = cid; t < T2; t += ncl) {
        const TileInfo ti = decode_pair(L, t, rank);
        const Problem& P = L.p[ti.pi];
        const int ohw = P.OH * P.OW, m0 = ti.tm * BM;
        for (int kb = 0; kb < ti.nkb; ++kb, ++g) {
          const int s = g % ST;
          if (g >= ST) umma::mbar_wait(&empty[s], ((g / ST) + 1) & 1);
          uint8_t* stage = smem + s * SB;
          const uint32_t fb = tc::mapa(&full[s], 0);
          const int kk = kb * BK;
          if (leader) umma::mbar_arrive_expect_tx(&full[s], 2u * SB);
          if (P.a_mode == 1) {
            tc::tma_load_2d_pair(stage, &L.tmA[ti.pi], kk, m0, fb);
          } else {
            const int img = m0 / ohw, rem = m0 - img * ohw;
            const int py = rem / P.OW, px = rem - py * P.OW;
            const int tap = kk / P.SC, c0 = kk - tap * P.SC;
            const int fr = tap / P.S, fs = tap - fr * P.S;
            if (MODE == FPROP)
              tc::tma_im2col_4d_pair(stage, &L.tmA[ti.pi], c0, px * P.stride - P.pad,
                                     py * P.stride - P.pad, img, (uint16_t)fs, (uint16_t)fr, fb);
            else
              tc::tma_im2col_4d_pair(stage, &L.tmA[ti.pi], c0, px + P.pad - (P.S - 1),
                                     py + P.pad - (P.R - 1), img, (uint16_t)(P.S - 1 - fs),
                                     (uint16_t)(P.R - 1 - fr), fb);
          }
          tc::tma_load_2d_pair(stage + 16384, &L.tm[ti.pi], kk,
                               P.brow0 + ti.tn * NT + rank * (NT / 2), fb);
        }
      }
    }
  } else if (warp == 4) {
    if (lane == 0 && leader) {  // ---- MMA issuer (leader only) ----
      const uint32_t idesc = tc::idesc_bf16(2 * BM, NT, false, false);
      const uint32_t sbase = tc::smem_u32(smem);
      int g = 0, it = 0;
      for (int t = cid; t < T2; t += ncl, ++it) {
        const TileInfo ti = decode_pair(L, t, 0);
        const int buf = it & 1;
        if (it >= 2) umma::mbar_wait(&tempty[buf], ((it >> 1) + 1) & 1);
        umma::fence_after();
        const uint32_t acc = tmem + (uint32_t)buf * bstride;
        for (int kb = 0; kb < ti.nkb; ++kb, ++g) {
          const int s = g % ST;
          umma::mbar_wait(&full[s], (g / ST) & 1);
          umma::fence_after();
          const uint32_t a_s = sbase + s * SB, b_s = a_s + 16384;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            tc::mma_bf16_pair(acc, tc::sdesc_sw128(a_s + ks * 32, 16, 1024),
                              tc::sdesc_sw128(b_s + ks * 32, 16, 1024), idesc,
                              (kb || ks) ? 1u : 0u);
          tc::commit_pair(&empty[s], (uint16_t)3);
        }
        tc::commit_pair(&tfull[buf], (uint16_t)3);
      }
    }
    __syncwarp();
  } else {  // ---- warps 0-3: epilogue (both CTAs) ----
    const uint32_t te0 = tc::mapa(&tempty[0], 0), te1 = tc::mapa(&tempty[1], 0);
    int it = 0;
    for (int t = cid; t < T2; t += ncl, ++it) {
      const TileInfo ti = decode_pair(L, t, rank);
      const int buf = it & 1;
      umma::mbar_wait(&tfull[buf], (it >> 1) & 1);
      umma::fence_after();
      epilogue<MODE>(L.p[ti.pi], tmem + (uint32_t)buf * bstride, warp, lane, ti.tm, ti.tn, 0,
                     ti.nkb, NT);
      umma::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_cluster(buf ? te1 : te0);
    }
  }
  umma::fence_before();
  __syncthreads();
  umma::cluster_sync();
  if (warp == 4) {
    umma::fence_after();
    tc::tmem_dealloc_pair(tmem, tcols);
  }
}

// ------------------------------------------------------------------------------
// Halo-tile variant for 3x3 stride-1 convolutions (FPROP on X, and DGRAD on dY
// with the rotated taps), input planes with C % 64 == 0.  An M tile is 128
// consecutive pixels of the PADDED output index o = y·(W+2) + x of one image
// (x >= W: junk rows the epilogue drops).  Per 64-channel block, ONE 4-D TMA box
// {64 ch, W+2 cols from x = -1, hrows rows from y = y0 - 1, 1 image} (zero fill
// outside the image) holds every input pixel the tile's nine taps touch, laid
// out as the same padded index; tap (r, s)'s A operand is that buffer shifted by
// x0 + r·(W+2) + s rows (the SW128 swizzle is address-based, so a shifted K-major
// descriptor is exact — tools/shift_test.cu).  TMA writes ≈ 1.3-2.3x the tile's
// pixels instead of the im2col 9x.  Two rings: halo buffers (2) and weight tiles
// (ST stages of NT x 64 K).  K order per output element: channel block outer, tap
// inner (for C == 64 that is the im2col kernels' k order; for C > 64 it differs
// from theirs) — fixed by the layer's shape, so packed == standalone bit for bit.
// ------------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(kThreads, 1) k_conv_gemm_halo(const __grid_constant__ Launch L) {
  static_assert(MODE != WGRAD, "halo variant: FPROP / DGRAD");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int NT = L.ntile, ST = L.stages;
  const uint32_t AB = (uint32_t)L.abytes, BB = (uint32_t)NT * 128u;
  uint8_t* abuf = smem;                       // 2 x AB
  uint8_t* bbuf = smem + 2 * AB;              // ST x BB
  uint64_t* bfull = reinterpret_cast<uint64_t*>(bbuf + ST * BB);
  uint64_t* bempty = bfull + ST;
  uint64_t* afull = bempty + ST;
  uint64_t* aempty = afull + 2;
  uint64_t* tfull = aempty + 2;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 160) {
    for (int s = 0; s < ST; ++s) {
      umma::mbar_init(&bfull[s], 1);
      umma::mbar_init(&bempty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      umma::mbar_init(&afull[b], 1);
      umma::mbar_init(&aempty[b], 1);
      umma::mbar_init(&tfull[b], 1);
      umma::mbar_init(&tempty[b], 128);
    }
    umma::mbar_fence_init();
  }
  const uint32_t tcols = umma::tmem_cols_pow2((uint32_t)(2 * NT));
  if (warp == 4) umma::tmem_alloc(tmem_slot, tcols);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 160) prefetch_b_panel<MODE>(L, blockIdx.x, L.ntile);

  tc::pdl_gate();
  const uint32_t bstride = tcols / 2;
  const int T = L.total_tiles;

  if (warp == 5) {
    if (lane == 0) {  // ---- TMA producer ----
      int g = 0, ga = 0;
      for (int t = blockIdx.x; t < T; t += gridDim.x) {
        const TileInfo ti = decode_tile(L, t, false);
        const Problem& P = L.p[ti.pi];
        const int img = ti.tm / P.tpi, o0 = (ti.tm - img * P.tpi) * BM;
        const int y0 = o0 / P.pw;
        const int ncb = P.SC / 64;
        for (int cb = 0; cb < ncb; ++cb, ++ga) {
          const int as = ga & 1;
          if (ga >= 2) umma::mbar_wait(&aempty[as], ((ga >> 1) + 1) & 1);
          umma::mbar_arrive_expect_tx(&afull[as], (uint32_t)(P.hrows * P.pw * 128));
          tc::tma_load_4d(abuf + as * AB, &L.tmA[ti.pi], cb * 64, -1, y0 - 1, img, &afull[as]);
          for (int tap = 0; tap < 9; ++tap, ++g) {
            const int s = g % ST;
            if (g >= ST) umma::mbar_wait(&bempty[s], ((g / ST) + 1) & 1);
            umma::mbar_arrive_expect_tx(&bfull[s], BB);
            tc::tma_load_2d(bbuf + s * BB, &L.tm[ti.pi], tap * P.SC + cb * 64,
                            P.brow0 + ti.tn * NT, &bfull[s]);
          }
        }
      }
    }
  } else if (warp == 4) {
    if (lane == 0) {  // ---- MMA issuer ----
      const uint32_t idesc = tc::idesc_bf16(BM, NT, false, false);
      const uint32_t abase = tc::smem_u32(abuf), bbase = tc::smem_u32(bbuf);
      int g = 0, ga = 0, it = 0;
      for (int t = blockIdx.x; t < T; t += gridDim.x, ++it) {
        const TileInfo ti = decode_tile(L, t, false);
        const Problem& P = L.p[ti.pi];
        const int img = ti.tm / P.tpi, o0 = (ti.tm - img * P.tpi) * BM;
        const int x0 = o0 - (o0 / P.pw) * P.pw;
        const int ncb = P.SC / 64;
        const int buf = it & 1;
        if (it >= 2) umma::mbar_wait(&tempty[buf], ((it >> 1) + 1) & 1);
        umma::fence_after();
        const uint32_t acc = tmem + (uint32_t)buf * bstride;
        for (int cb = 0; cb < ncb; ++cb, ++ga) {
          const int as = ga & 1;
          umma::mbar_wait(&afull[as], (ga >> 1) & 1);
          umma::fence_after();
          for (int tap = 0; tap < 9; ++tap, ++g) {
            const int s = g % ST;
            umma::mbar_wait(&bfull[s], (g / ST) & 1);
            umma::fence_after();
            const int r = tap / 3, q = tap - 3 * r;
            const int off = MODE == FPROP ? x0 + r * P.pw + q : x0 + (2 - r) * P.pw + (2 - q);
            const uint32_t a_s = abase + as * AB + (uint32_t)off * 128u, b_s = bbase + s * BB;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
              tc::mma_bf16(acc, tc::sdesc_sw128(a_s + ks * 32, 16, 1024),
                           tc::sdesc_sw128(b_s + ks * 32, 16, 1024), idesc,
                           (cb || tap || ks) ? 1u : 0u);
            umma::commit(&bempty[s]);
          }
          umma::commit(&aempty[as]);
        }
        umma::commit(&tfull[buf]);
      }
    }
    __syncwarp();
  } else {  // ---- warps 0-3: epilogue ----
    int it = 0;
    for (int t = blockIdx.x; t < T; t += gridDim.x, ++it) {
      const TileInfo ti = decode_tile(L, t, false);
      const int buf = it & 1;
      umma::mbar_wait(&tfull[buf], (it >> 1) & 1);
      umma::fence_after();
      epilogue<MODE>(L.p[ti.pi], tmem + (uint32_t)buf * bstride, warp, lane, ti.tm, ti.tn, 0, 1,
                     NT);
      umma::fence_before();
      tc::mbar_arrive(&tempty[buf]);
    }
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 4) {
    umma::fence_after();
    umma::tmem_dealloc(tmem, tcols);
  }
}

// ------------------------------------------------------------------------------
// Weights-resident halo variant (C == 64, N tile <= 64: ResNet's 56x56x64 layers).
// The nine 64-deep weight tiles of a problem (9 x NT x 128 B <= 72 KB) are loaded
// once per problem into shared memory; a CTA owns a CONTIGUOUS range of tiles
// (mostly one problem) and per tile waits for one halo box only, then issues its
// 36 MMAs back to back — no per-tap barrier round trips for these short MMAs.
// Same tap order and operands as k_conv_gemm_halo: identical results.
// ------------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(kThreads, 1) k_conv_gemm_halo_res(const __grid_constant__ Launch L) {
  static_assert(MODE != WGRAD, "halo variant: FPROP / DGRAD");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int NT = L.ntile;
  const uint32_t AB = (uint32_t)L.abytes, BB = (uint32_t)NT * 128u;
  uint8_t* abuf = smem;                 // 2 x AB halo buffers
  uint8_t* bres = smem + 2 * AB;        // 9 x BB resident weight tiles
  uint64_t* afull = reinterpret_cast<uint64_t*>(bres + 9 * BB);
  uint64_t* aempty = afull + 2;
  uint64_t* tfull = aempty + 2;
  uint64_t* tempty = tfull + 2;
  uint64_t* wfull = tempty + 2;
  uint64_t* wempty = wfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wempty + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 160) {
    for (int b = 0; b < 2; ++b) {
      umma::mbar_init(&afull[b], 1);
      umma::mbar_init(&aempty[b], 1);
      umma::mbar_init(&tfull[b], 1);
      umma::mbar_init(&tempty[b], 128);
    }
    umma::mbar_init(wfull, 1);
    umma::mbar_init(wempty, 1);
    umma::mbar_fence_init();
  }
  const uint32_t tcols = umma::tmem_cols_pow2((uint32_t)(2 * NT));
  if (warp == 4) umma::tmem_alloc(tmem_slot, tcols);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 160) prefetch_b_panel<MODE>(L, blockIdx.x, L.ntile);

  tc::pdl_gate();
  const uint32_t bstride = tcols / 2;
  const int T = L.total_tiles, G = gridDim.x;
  const int t0 = (int)((long long)T * blockIdx.x / G), t1 = (int)((long long)T * (blockIdx.x + 1) / G);

  if (warp == 5) {
    if (lane == 0) {  // ---- TMA producer ----
      int ga = 0, cur = -1, nw = 0;
      for (int t = t0; t < t1; ++t, ++ga) {
        const TileInfo ti = decode_tile(L, t, false);
        const Problem& P = L.p[ti.pi];
        if (ti.pi != cur) {  // this problem's weights (after the previous ones are used)
          if (nw > 0) umma::mbar_wait(wempty, (nw - 1) & 1);
          umma::mbar_arrive_expect_tx(wfull, 9u * BB);
          for (int tap = 0; tap < 9; ++tap)
            tc::tma_load_2d(bres + tap * BB, &L.tm[ti.pi], tap * 64, P.brow0 + ti.tn * NT, wfull);
          cur = ti.pi;
          ++nw;
        }
        const int img = ti.tm / P.tpi, o0 = (ti.tm - img * P.tpi) * BM;
        const int as = ga & 1;
        if (ga >= 2) umma::mbar_wait(&aempty[as], ((ga >> 1) + 1) & 1);
        umma::mbar_arrive_expect_tx(&afull[as], (uint32_t)(P.hrows * P.pw * 128));
        tc::tma_load_4d(abuf + as * AB, &L.tmA[ti.pi], 0, -1, o0 / P.pw - 1, img, &afull[as]);
      }
    }
  } else if (warp == 4) {
    if (lane == 0) {  // ---- MMA issuer ----
      const uint32_t idesc = tc::idesc_bf16(BM, NT, false, false);
      const uint32_t abase = tc::smem_u32(abuf), bbase = tc::smem_u32(bres);
      int ga = 0, it = 0, cur = -1, nw = 0;
      for (int t = t0; t < t1; ++t, ++ga, ++it) {
        const TileInfo ti = decode_tile(L, t, false);
        const Problem& P = L.p[ti.pi];
        if (ti.pi != cur) {
          umma::mbar_wait(wfull, nw & 1);
          cur = ti.pi;
          ++nw;
        }
        const int img = ti.tm / P.tpi, o0 = (ti.tm - img * P.tpi) * BM;
        const int x0 = o0 - (o0 / P.pw) * P.pw;
        const int buf = it & 1, as = ga & 1;
        if (it >= 2) umma::mbar_wait(&tempty[buf], ((it >> 1) + 1) & 1);
        umma::mbar_wait(&afull[as], (ga >> 1) & 1);
        umma::fence_after();
        const uint32_t acc = tmem + (uint32_t)buf * bstride;
        for (int tap = 0; tap < 9; ++tap) {
          const int r = tap / 3, q = tap - 3 * r;
          const int off = MODE == FPROP ? x0 + r * P.pw + q : x0 + (2 - r) * P.pw + (2 - q);
          const uint32_t a_s = abase + as * AB + (uint32_t)off * 128u, b_s = bbase + tap * BB;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            tc::mma_bf16(acc, tc::sdesc_sw128(a_s + ks * 32, 16, 1024),
                         tc::sdesc_sw128(b_s + ks * 32, 16, 1024), idesc,
                         (tap || ks) ? 1u : 0u);
        }
        umma::commit(&aempty[as]);
        umma::commit(&tfull[buf]);
        // last tile of this problem in the range: its weights may be replaced
        if (t + 1 >= t1 || decode_tile(L, t + 1, false).pi != cur) umma::commit(wempty);
      }
    }
    __syncwarp();
  } else {  // ---- warps 0-3: epilogue ----
    int it = 0;
    for (int t = t0; t < t1; ++t, ++it) {
      const TileInfo ti = decode_tile(L, t, false);
      const int buf = it & 1;
      umma::mbar_wait(&tfull[buf], (it >> 1) & 1);
      umma::fence_after();
      epilogue<MODE>(L.p[ti.pi], tmem + (uint32_t)buf * bstride, warp, lane, ti.tm, ti.tn, 0, 1,
                     NT);
      umma::fence_before();
      tc::mbar_arrive(&tempty[buf]);
    }
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 4) {
    umma::fence_after();
    umma::tmem_dealloc(tmem, tcols);
  }
}

}  // namespace cg
