// pk_cnn.cu — conv pack runtime behind the packtrain_b200.h C-ABI (pk_cnet_*).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "packtrain_b200.h"
#include "pk_convgemm.cuh"
#include "pk_cnn_ops.cuh"

namespace {

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

bool encode_fn() {
  std::call_once(g_encode_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode != nullptr;
}

PFN_cuTensorMapEncodeIm2col_v12000 g_encode_i2c = nullptr;
std::once_flag g_i2c_once;
int g_driver_version = 0;

// 4-D NHWC bf16 im2col map (dims {c, w, h, n}, pixel pitch `ld` elements):
// boxes of `pixels` GEMM rows x 64 channels, SW128, zero fill outside the image.
// lower/upper: the pixel box corners {w, h} (CUTLASS sm100 conv conventions).
bool make_map_im2col(CUtensorMap* m, const void* base, int n, int h, int w, int c, int ld,
                     int lower_w, int lower_h, int upper_w, int upper_h, int stride,
                     int pixels, int chans = 64) {
  std::call_once(g_i2c_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode_i2c = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(fn);
    cudaDriverGetVersion(&g_driver_version);
  });
  if (!g_encode_i2c) return false;
  cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
  cuuint64_t strides[3] = {(cuuint64_t)ld * 2, (cuuint64_t)w * ld * 2,
                           (cuuint64_t)h * w * ld * 2};
  int lower[2] = {lower_w, lower_h}, upper[2] = {upper_w, upper_h};
  cuuint32_t es[4] = {1, (cuuint32_t)stride, (cuuint32_t)stride, 1};
  if (g_encode_i2c(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides,
                   lower, upper, (cuuint32_t)chans, (cuuint32_t)pixels, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   chans == 16 ? CU_TENSOR_MAP_SWIZZLE_32B
                               : (chans == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B),
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  // the driver workaround CUTLASS applies to im2col maps of tensors < 128 KiB on
  // drivers <= 13.1 (cute/atom/copy_traits_sm90_im2col.hpp)
  const double bytes = (double)n * h * w * ld * 2;
  if (g_driver_version <= 13010 && bytes < 131072.0)
    reinterpret_cast<uint64_t*>(m)[1] &= ~(1ull << 21);
  return true;
}

// 2-D bf16 tensor map [rows][cols] (row pitch `ld` elements), box {box_cols, box_rows},
// SW128 for 64-column boxes, SW32 for 16-column boxes
bool make_map_2d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                 uint32_t box_rows, uint32_t box_cols = 64) {
  if (!encode_fn()) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  return g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  box_cols == 16 ? CU_TENSOR_MAP_SWIZZLE_32B
                                 : (box_cols == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                   : CU_TENSOR_MAP_SWIZZLE_128B),
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 3-D bf16 tensor map [depth][rows][cols] (row pitch `ld`, depth pitch `dstride`
// elements), box {64 cols, box_rows, 1}, SW128
bool make_map_3d(CUtensorMap* m, const void* base, uint64_t depth, uint64_t rows, uint64_t cols,
                 uint64_t ld, uint64_t dstride, uint32_t box_rows) {
  if (!encode_fn()) return false;
  cuuint64_t dims[3] = {cols, rows, depth};
  cuuint64_t strides[2] = {ld * 2, dstride * 2};
  cuuint32_t box[3] = {64, box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }
inline int rup(int a, int b) { return (a + b - 1) / b * b; }

// fill tile counts / prefix and launch one grouped implicit-GEMM conv
template <int MODE>
cudaError_t launch_gemm(cg::Launch& L, cudaStream_t st) {
  static bool attr_set = false;
  int tiles = 0;
  for (int i = 0; i < L.nprob; ++i) {
    cg::Problem& p = L.p[i];
    p.tiles_m = cdiv(p.M, cg::BM);
    p.tiles_n = cdiv(p.N, L.ntile);
    if (MODE != cg::WGRAD) p.splits = 1;
    p.tile0 = tiles;
    tiles += p.tiles_m * p.tiles_n * p.splits;
  }
  L.total_tiles = tiles;
  if (tiles == 0) return cudaSuccess;
  const size_t smem = cg::smem_bytes(L.ntile, L.stages);
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(cg::k_conv_gemm<MODE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  cg::k_conv_gemm<MODE><<<tiles, cg::kThreads, smem, st>>>(L);
  return cudaGetLastError();
}


thread_local std::string g_err;
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

size_t prob_size(int kind) {
  switch (kind) {
    case PK_CNN_CONV_FPROP:
    case PK_CNN_CONV_DGRAD:
    case PK_CNN_CONV_WGRAD: return sizeof(pk_cnn_conv);
    case PK_CNN_BN_STATS:
    case PK_CNN_BN_APPLY:
    case PK_CNN_BN_BWD_REDUCE:
    case PK_CNN_BN_BWD_APPLY: return sizeof(pk_cnn_bn);
    case PK_CNN_DW_FPROP:
    case PK_CNN_DW_DGRAD:
    case PK_CNN_DW_WGRAD: return sizeof(pk_cnn_dw);
    case PK_CNN_MAXPOOL_FWD:
    case PK_CNN_MAXPOOL_BWD:
    case PK_CNN_AVGPOOL_FWD:
    case PK_CNN_AVGPOOL_BWD: return sizeof(pk_cnn_pool);
    case PK_CNN_XENT: return sizeof(pk_cnn_head);
    case PK_CNN_BIAS_ACT_BWD: return sizeof(pk_cnn_bias);
    case PK_CNN_SPLIT_REDUCE: return sizeof(pk_cnn_reduce);
    case PK_CNN_OPT: return sizeof(pk_cnn_opt_seg);
    case PK_CNN_PUBLISH_T: return sizeof(pk_cnn_tpose);
    case PK_CNN_COMMIT: return sizeof(pk_cnn_commit);
    case PK_CNN_GATHER: return sizeof(pk_cnn_gather);
    case PK_CNN_IM2COL: return sizeof(pk_cnn_im2col);
  }
  return 0;
}

long long items(long long rows, int c) { return rows * (c / 8); }
int cgp_of(int c) {  // channel groups rounded up to a power of two (cnn::lanes_of)
  int g = 1;
  while (g < c / 8) g <<= 1;
  return g;
}
int blocks_of(long long n) { return (int)((n + cnn::kBlock - 1) / cnn::kBlock); }

// blocks one problem of a non-conv kind needs
int prob_blocks(int kind, const void* pr) {
  switch (kind) {
    case PK_CNN_BN_STATS:
    case PK_CNN_BN_BWD_REDUCE: {
      const pk_cnn_bn& P = *static_cast<const pk_cnn_bn*>(pr);
      return cdiv(P.rows, P.rpb);
    }
    case PK_CNN_BN_APPLY:
    case PK_CNN_BN_BWD_APPLY: {
      const pk_cnn_bn& P = *static_cast<const pk_cnn_bn*>(pr);
      return cnn::apply_blocks(P.rows, P.c, P.pad0);
    }
    case PK_CNN_DW_FPROP:
    case PK_CNN_DW_DGRAD: {
      const pk_cnn_dw& P = *static_cast<const pk_cnn_dw*>(pr);
      const int oh = kind == PK_CNN_DW_FPROP ? P.p : P.h, ow = kind == PK_CNN_DW_FPROP ? P.q : P.w;
      if (cnn::dw_strip_ok(P))  // output strips of dw_strip_xs pixels
        return blocks_of(items((long long)P.n * oh * cdiv(ow, cnn::dw_strip_xs(kind, P.stride)),
                               P.c));
      return blocks_of(items((long long)P.n * oh * ow, P.c));
    }
    case PK_CNN_DW_WGRAD: {
      const pk_cnn_dw& P = *static_cast<const pk_cnn_dw*>(pr);
      const int splits = cdiv((long long)P.n * P.p * P.q, P.ppb);
      return cnn::dw_fast(P, kind) ? splits * cnn::dw_wgrad_chunks(P.c) : splits;
    }
    case PK_CNN_MAXPOOL_FWD: {
      const pk_cnn_pool& P = *static_cast<const pk_cnn_pool*>(pr);
      return blocks_of(items((long long)P.n * P.p * P.q, P.c));
    }
    case PK_CNN_AVGPOOL_FWD: {
      const pk_cnn_pool& P = *static_cast<const pk_cnn_pool*>(pr);
      const bool global = P.r == P.h && P.s == P.w && P.pad == 0 && P.p == 1 && P.q == 1;
      return blocks_of(items((long long)P.n * P.p * P.q, P.c) *
                       (global ? cnn::avgpool_lanes(P.h * P.w) : 1));
    }
    case PK_CNN_MAXPOOL_BWD:
    case PK_CNN_AVGPOOL_BWD: {
      const pk_cnn_pool& P = *static_cast<const pk_cnn_pool*>(pr);
      return blocks_of(items((long long)P.n * P.h * P.w, P.c));
    }
    case PK_CNN_BIAS_ACT_BWD: {
      const pk_cnn_bias& P = *static_cast<const pk_cnn_bias*>(pr);
      return cdiv(P.rows, P.rpb);
    }
    case PK_CNN_SPLIT_REDUCE: {
      const pk_cnn_reduce& P = *static_cast<const pk_cnn_reduce*>(pr);
      return blocks_of((P.len + 3) / 4);
    }
    case PK_CNN_OPT: {
      const pk_cnn_opt_seg& P = *static_cast<const pk_cnn_opt_seg*>(pr);
      return (int)((P.len + cnn::kOptChunk - 1) / cnn::kOptChunk);
    }
    case PK_CNN_PUBLISH_T: {
      const pk_cnn_tpose& P = *static_cast<const pk_cnn_tpose*>(pr);
      return P.taps * cdiv(P.k, cnn::kTposeTile) * cdiv(P.c, cnn::kTposeTile);
    }
    case PK_CNN_GATHER: {
      const pk_cnn_gather& P = *static_cast<const pk_cnn_gather*>(pr);
      return (int)((P.row_bytes * P.rows + cnn::kGatherChunk - 1) / cnn::kGatherChunk);
    }
    case PK_CNN_IM2COL: {
      const pk_cnn_im2col& P = *static_cast<const pk_cnn_im2col*>(pr);
      return P.n * P.p * cdiv(P.q, cnn::kIm2colPix);  // runs of an output row
    }
  }
  return 0;
}

int head_blocks(int, const void*) { return 1; }  // XENT: one block per member

std::string check_prob(int kind, const void* pr) {
  auto c8 = [](int c) { return c > 0 && c % 8 == 0 && c <= 2048; };
  switch (kind) {
    case PK_CNN_BN_STATS:
    case PK_CNN_BN_APPLY:
    case PK_CNN_BN_BWD_REDUCE:
    case PK_CNN_BN_BWD_APPLY: {
      const pk_cnn_bn& P = *static_cast<const pk_cnn_bn*>(pr);
      if (!c8(P.c) || P.rows <= 0) return "bn: channels must be a multiple of 8 in [8, 2048]";
      if ((kind == PK_CNN_BN_STATS || kind == PK_CNN_BN_BWD_REDUCE) &&
          (P.rpb < 1 || P.rpb % 32 || cdiv(P.rows, P.rpb) > cnn::kRedMaxBlocks))
        return "bn: rows per block must be a positive multiple of 32, <= 256 blocks";
      break;
    }
    case PK_CNN_DW_FPROP:
    case PK_CNN_DW_DGRAD:
    case PK_CNN_DW_WGRAD: {
      const pk_cnn_dw& P = *static_cast<const pk_cnn_dw*>(pr);
      if (!c8(P.c) || P.r * P.s > 9 || P.stride < 1) return "dw: c % 8, r*s <= 9";
      if (kind == PK_CNN_DW_WGRAD && P.ppb < 1) return "dw: pixels per block >= 1";
      if (kind == PK_CNN_DW_WGRAD && cnn::dw_fast(P, kind) && P.ppb % cnn::dw_wgrad_lanes(P.c))
        return "dw: 3x3 WGRAD pixels per block must be a multiple of the pixel lanes";
      if (kind == PK_CNN_DW_WGRAD && prob_blocks(kind, pr) > cnn::kRedMaxBlocks)
        return "dw: WGRAD <= 256 blocks (channel chunks x pixel splits)";
      break;
    }
    case PK_CNN_MAXPOOL_FWD:
    case PK_CNN_MAXPOOL_BWD:
    case PK_CNN_AVGPOOL_FWD:
    case PK_CNN_AVGPOOL_BWD: {
      const pk_cnn_pool& P = *static_cast<const pk_cnn_pool*>(pr);
      if (P.c % 8 || P.r * P.s > 255 || P.stride < 1) return "pool: c % 8, window <= 255";
      if ((long long)P.n * std::max(P.h * P.w, P.p * P.q) * (P.c / 8) >= (1LL << 31))
        return "pool: n*h*w*c/8 must stay below 2^31";
      break;
    }
    case PK_CNN_BIAS_ACT_BWD: {
      const pk_cnn_bias& P = *static_cast<const pk_cnn_bias*>(pr);
      if (!c8(P.c) || P.rpb < 1 || cdiv(P.rows, P.rpb) > cnn::kRedMaxBlocks)
        return "bias: channels % 8 in [8, 2048], <= 256 row blocks";
      break;
    }
    case PK_CNN_XENT: {
      const pk_cnn_head& P = *static_cast<const pk_cnn_head*>(pr);
      if (P.rows <= 0 || P.rows > 4096 || P.classes <= 0 || P.ldl < P.classes)
        return "xent: 0 < rows <= 4096, classes <= ldl";
      break;
    }
    case PK_CNN_SPLIT_REDUCE: {
      const pk_cnn_reduce& P = *static_cast<const pk_cnn_reduce*>(pr);
      if (P.len % 4 || P.splits < 1) return "split_reduce: len % 4";
      break;
    }
    case PK_CNN_GATHER: {
      const pk_cnn_gather& P = *static_cast<const pk_cnn_gather*>(pr);
      if (P.row_bytes % 16 || P.rows < 0) return "gather: row_bytes % 16";
      break;
    }
    case PK_CNN_IM2COL: {
      const pk_cnn_im2col& P = *static_cast<const pk_cnn_im2col*>(pr);
      if (P.ldo % 8 || P.ldo > 256 || P.cp % 8 || P.c < 1 || P.c > 8 || P.c > P.cp ||
          P.r * P.s * P.c > P.ldo ||
          P.r * cnn::im2col_stage_cols(P.s, P.stride) > cnn::kIm2colStage ||
          P.stride < 1 || (long long)P.n * P.p * P.q * (P.ldo / 8) >= (1LL << 31))
        return "im2col: ldo <= 256, ldo and cp multiples of 8, r*s*c <= ldo, c <= min(cp, 8), "
               "r*(63*stride+s) <= 1024";
      break;
    }
  }
  return std::string();
}

struct OpRec {
  int kind = 0, nprob = 0, nblocks = 0, lane = 0;
  int ntile = 0, stages = 0;
  size_t probs_off = 0, blk_off = 0;  // offsets into the device descriptor block (OPT, COMMIT)
  std::vector<cg::Launch> conv;       // conv ops: launches of <= kMaxProblems problems
  // other kinds: parameter packs of <= cnn::kPack problems (raw cnn::Pack<T> bytes)
  std::vector<std::vector<uint8_t>> packs;
  std::vector<int> pack_blocks;
};

// split one op's problems into kernel-parameter packs of <= kPack problems
template <class T>
void make_packs(OpRec& r, const T* pr, int n, int (*blocks)(int, const void*)) {
  for (int i0 = 0; i0 < n; i0 += cnn::kPack) {
    cnn::Pack<T> P;
    memset(&P, 0, sizeof(P));
    P.nprob = std::min(cnn::kPack, n - i0);
    for (int j = 0; j < P.nprob; ++j) {
      P.p[j] = pr[i0 + j];
      if constexpr (std::is_same<T, pk_cnn_bn>::value) {
        // BN apply kinds: about two waves of blocks for the whole launch (the row
        // tiles of larger layers are looped over; an elementwise partition)
        if (r.kind == PK_CNN_BN_APPLY || r.kind == PK_CNN_BN_BWD_APPLY)
          P.p[j].pad0 = std::max(16, 2 * 148 * 3 / P.nprob);
      }
      P.blk0[j + 1] = P.blk0[j] + blocks(r.kind, &P.p[j]);
    }
    std::vector<uint8_t> raw(sizeof(P));
    memcpy(raw.data(), &P, sizeof(P));
    r.packs.push_back(std::move(raw));
    r.pack_blocks.push_back(P.blk0[P.nprob]);
  }
}

}  // namespace

constexpr int kMaxLanes = 8;

struct pk_cnn_prog {
  int device = 0;
  std::vector<OpRec> ops;
  cudaStream_t lane_st[kMaxLanes + 1] = {};  // side streams of lanes 1..kMaxLanes
  cudaEvent_t fork_ev = nullptr, join_ev[kMaxLanes + 1] = {};
  // async lanes (op lane 16 + a): ops that only feed the end of the step (weight
  // gradients) run on these, each forking from the program stream where it sits
  cudaStream_t async_st[kMaxLanes + 1] = {};
  cudaEvent_t async_fork[kMaxLanes + 1] = {}, async_join[kMaxLanes + 1] = {};
  uint8_t* dmem = nullptr;
  int launches = 0;
  cudaGraphExec_t gexec = nullptr;
  cudaStream_t gstream = nullptr;
};

namespace {

// stride-2 DGRAD of a 3x3 pad-1 or 1x1 pad-0 conv on even planes runs as four
// stride-1 problems, one per dX parity class (a, b) = (y & 1, x & 1): class pixels
// (2i + a, 2j + b) read dY at (i + dr, j + ds) for the taps (r, s) with r ≡ a + pad,
// s ≡ b + pad (mod 2) — no zero taps reach the tensor cores (a 3x3 class has 1, 2
// or 4 taps; a 1x1 conv's odd classes have none and write zeros / keep the sum)
bool dgrad_parity(const pk_cnn_conv& g) {
  return g.stride == 2 && g.h == 2 * g.p && g.w == 2 * g.q && g.k % 64 == 0 &&
         ((g.r == 3 && g.s == 3 && g.pad == 1) || (g.r == 1 && g.s == 1 && g.pad == 0));
}

int conv_to_launches(int kind, const pk_cnn_conv* pr0, int n0, int ntile, int stages,
                     std::vector<cg::Launch>& out) {
  // (problem, parity class or -1) items; parity DGRADs expand to four
  std::vector<pk_cnn_conv> exp;
  std::vector<int> cls;
  for (int i = 0; i < n0; ++i) {
    if (kind == PK_CNN_CONV_DGRAD && dgrad_parity(pr0[i])) {
      // a 1x1 conv's odd classes have no tap: needed only to write zeros
      const int ncls = pr0[i].r == 1 && pr0[i].accumulate ? 1 : 4;
      for (int c = 0; c < ncls; ++c) {
        exp.push_back(pr0[i]);
        cls.push_back(c);
      }
    } else {
      exp.push_back(pr0[i]);
      cls.push_back(-1);
    }
  }
  const pk_cnn_conv* pr = exp.data();
  const int n = (int)exp.size();
  for (int i0 = 0; i0 < n; i0 += cg::kMaxProblems) {
    cg::Launch L;
    memset(&L, 0, sizeof(L));
    L.nprob = std::min(cg::kMaxProblems, n - i0);
    L.ntile = ntile;
    L.stages = stages;
    int tiles = 0;
    for (int j = 0; j < L.nprob; ++j) {
      const pk_cnn_conv& g = pr[i0 + j];
      cg::Problem& p = L.p[j];
      p.par = cls[i0 + j];
      if (g.c % 8 || g.k % 8 || (g.stride != 1 && g.stride != 2))
        return fail(PK_ERR_ARG, "conv: c, k multiples of 8; stride 1 or 2");
      p.R = g.r; p.S = g.s; p.stride = g.stride; p.pad = g.pad;
      p.dst = g.dst;
      const bool one = g.r == 1 && g.s == 1 && g.stride == 1 && g.pad == 0;
      if (kind == PK_CNN_CONV_FPROP) {
        const int kpad = rup(g.r * g.s * g.c, 64);
        if (!g.idx && one) {
          p.a_mode = 1;
          if (!make_map_2d(&L.tmA[j], g.src, (uint64_t)g.n * g.h * g.w, g.c, g.ldx, cg::BM))
            return fail(PK_ERR_CUDA, "conv: FPROP activation map");
        } else if (!g.idx && g.c % 64 == 0) {
          p.a_mode = 2;
          if (!make_map_im2col(&L.tmA[j], g.src, g.n, g.h, g.w, g.c, g.ldx, -g.pad, -g.pad,
                               g.pad - (g.s - 1), g.pad - (g.r - 1), g.stride, cg::BM))
            return fail(PK_ERR_CUDA, "conv: FPROP im2col map");
        } else if (!g.idx && g.c == 16 && g.ldx == 16 && g.r * g.s <= 255) {
          p.a_mode = 3;  // 16-channel input: one tap per 16-deep K chunk, SW32
          if (!make_map_im2col(&L.tmA[j], g.src, g.n, g.h, g.w, 16, 16, -g.pad, -g.pad,
                               g.pad - (g.s - 1), g.pad - (g.r - 1), g.stride, cg::BM, 16))
            return fail(PK_ERR_CUDA, "conv: FPROP 16-channel im2col map");
        }
        p.src = static_cast<const __nv_bfloat16*>(g.src);
        p.idx = reinterpret_cast<const long long*>(g.idx);
        p.bias = g.bias; p.act = g.act; p.out_f32 = g.out_f32;
        p.nseg = g.nseg; p.dseg = g.dseg;
        p.M = g.n * g.p * g.q; p.N = g.k; p.K = g.r * g.s * g.c;
        p.SH = g.h; p.SW = g.w; p.SC = g.c; p.sld = g.ldx;
        p.OH = g.p; p.OW = g.q; p.dld = g.ldo;
        if (!make_map_2d(&L.tm[j], g.wt, g.k, kpad, kpad, ntile, p.a_mode == 3 ? 16 : 64))
          return fail(PK_ERR_CUDA, "conv: cuTensorMapEncodeTiled failed (FPROP weights)");
        p.wbase = static_cast<const uint8_t*>(g.wt);
        p.wpitch = kpad * 2;
        p.splits = 1;
      } else if (kind == PK_CNN_CONV_DGRAD && p.par >= 0) {
        const int kpadt = rup(g.r * g.s * g.k, 64);
        const int a = p.par >> 1, b = p.par & 1;
        p.ntap = 0;
        for (int r = 0; r < g.r; ++r)
          for (int q = 0; q < g.s; ++q)
            if (((a + g.pad - r) & 1) == 0 && ((b + g.pad - q) & 1) == 0) {
              p.tapk[p.ntap] = r * g.s + q;
              p.tdr[p.ntap] = (a + g.pad - r) / 2;
              p.tds[p.ntap] = (b + g.pad - q) / 2;
              ++p.ntap;
            }
        if (g.r == 1) {  // 1x1: class (0, 0) is a plain GEMM over dY rows, the rest K = 0
          p.a_mode = 1;
          if (!make_map_2d(&L.tmA[j], g.src, (uint64_t)g.n * g.p * g.q, g.k, g.ldy, cg::BM))
            return fail(PK_ERR_CUDA, "conv: DGRAD parity activation map");
        } else {  // 3x3: dY windows (i + {0,1}, j + {0,1}), zero fill past the plane
          p.a_mode = 5;
          if (!make_map_im2col(&L.tmA[j], g.src, g.n, g.p, g.q, g.k, g.ldy, 0, 0, 0, 0, 1,
                               cg::BM))
            return fail(PK_ERR_CUDA, "conv: DGRAD parity im2col map");
        }
        p.src = static_cast<const __nv_bfloat16*>(g.src);
        p.accumulate = g.accumulate;
        p.M = g.n * g.p * g.q; p.N = g.c; p.K = p.ntap * g.k;
        p.SH = g.p; p.SW = g.q; p.SC = g.k; p.sld = g.ldy;
        p.OH = g.p; p.OW = g.q; p.dld = g.ldo;
        p.DH = g.h; p.DW = g.w;
        if (!make_map_2d(&L.tm[j], g.wt, g.c, kpadt, kpadt, ntile))
          return fail(PK_ERR_CUDA, "conv: cuTensorMapEncodeTiled failed (DGRAD weights)");
        p.wbase = static_cast<const uint8_t*>(g.wt);
        p.wpitch = kpadt * 2;
        p.splits = 1;
      } else if (kind == PK_CNN_CONV_DGRAD) {
        const int kpadt = rup(g.r * g.s * g.k, 64);
        if (one) {
          p.a_mode = 1;
          if (!make_map_2d(&L.tmA[j], g.src, (uint64_t)g.n * g.p * g.q, g.k, g.ldy, cg::BM))
            return fail(PK_ERR_CUDA, "conv: DGRAD activation map");
        } else if (g.stride == 1 && g.k % 64 == 0) {
          p.a_mode = 2;
          if (!make_map_im2col(&L.tmA[j], g.src, g.n, g.p, g.q, g.k, g.ldy, g.pad - (g.s - 1),
                               g.pad - (g.r - 1), g.pad - (g.s - 1) + g.w - g.q,
                               g.pad - (g.r - 1) + g.h - g.p, 1, cg::BM))
            return fail(PK_ERR_CUDA, "conv: DGRAD im2col map");
        } else if (g.stride == 1 && g.k == 32 && g.ldy % 8 == 0) {
          // 32-channel dY (DenseNet growth convs): two taps per 64-deep k-block, each
          // a 128-pixel x 32-channel SW64 im2col box (cg::Problem a_mode 6)
          p.a_mode = 6;
          if (!make_map_im2col(&L.tmA[j], g.src, g.n, g.p, g.q, 32, g.ldy, g.pad - (g.s - 1),
                               g.pad - (g.r - 1), g.pad - (g.s - 1) + g.w - g.q,
                               g.pad - (g.r - 1) + g.h - g.p, 1, cg::BM, 32))
            return fail(PK_ERR_CUDA, "conv: DGRAD 32-channel im2col map");
        }
        p.src = static_cast<const __nv_bfloat16*>(g.src);
        p.accumulate = g.accumulate;
        p.M = g.n * g.h * g.w; p.N = g.c; p.K = g.r * g.s * g.k;
        p.SH = g.p; p.SW = g.q; p.SC = g.k; p.sld = g.ldy;
        p.OH = g.h; p.OW = g.w; p.dld = g.ldo;
        if (!make_map_2d(&L.tm[j], g.wt, g.c, kpadt, kpadt, ntile, p.a_mode == 6 ? 32 : 64))
          return fail(PK_ERR_CUDA, "conv: cuTensorMapEncodeTiled failed (DGRAD weights)");
        p.wbase = static_cast<const uint8_t*>(g.wt);
        p.wpitch = kpadt * 2;
        p.splits = 1;
      } else {
        if (ntile % 64) return fail(PK_ERR_ARG, "conv: WGRAD N tile must be a multiple of 64");
        const int kpad = rup(g.r * g.s * g.c, 64);
        const int pix = g.n * g.p * g.q;
        p.src = static_cast<const __nv_bfloat16*>(g.src);
        p.src2 = static_cast<const __nv_bfloat16*>(g.dy);
        p.idx = reinterpret_cast<const long long*>(g.idx);
        p.M = g.k; p.N = g.r * g.s * g.c; p.K = pix;
        const int sp = std::max(1, g.splits);
        p.kper = rup(cdiv(pix, sp), 64);
        p.splits = cdiv(pix, p.kper);
        if (p.splits != sp) return fail(PK_ERR_ARG, "conv: WGRAD splits leave an empty split");
        p.flag = p.splits == 1 ? g.flag : nullptr;
        const bool c16 = g.c == 16 && g.ldx == 16 && !one;
        if (!g.idx && (one || g.c % 64 == 0 || c16)) {
          p.b_mode = one ? 1 : (c16 ? 3 : 2);
          const bool ok =
              one ? make_map_2d(&L.tm[j], g.src, (uint64_t)g.n * g.h * g.w, g.c, g.ldx, 64)
                  : make_map_im2col(&L.tm[j], g.src, g.n, g.h, g.w, g.c, g.ldx, -g.pad, -g.pad,
                                    g.pad - (g.s - 1), g.pad - (g.r - 1), g.stride, 64,
                                    c16 ? 16 : 64);
          if (g.nseg > 0) {  // members concatenated along N (shared-input first layer)
            if (g.nseg != 64 || g.k % 64 || p.splits < 2)
              return fail(PK_ERR_ARG, "conv: concatenated WGRAD needs 64 channels per member "
                                      "and pixel splits");
            if (!ok || !make_map_3d(&L.tmA[j], g.dy, (uint64_t)(g.k / 64), (uint64_t)pix, 64,
                                    g.ldy, (uint64_t)g.dseg, 64))
              return fail(PK_ERR_CUDA, "conv: WGRAD operand maps");
            p.swap = 1;
            p.wseg = 64;
            p.M = g.r * g.s * g.c;
            p.N = g.k;
          } else {
            if (!ok || !make_map_2d(&L.tmA[j], g.dy, (uint64_t)pix, g.k, g.ldy, 64))
              return fail(PK_ERR_CUDA, "conv: WGRAD operand maps");
            if (g.k <= 64 && ntile == 64) {  // swapped orientation (see cg::Problem::swap)
              p.swap = 1;
              p.M = g.r * g.s * g.c;
              p.N = g.k;
            }
          }
        } else if (g.nseg > 0) {
          return fail(PK_ERR_ARG, "conv: concatenated WGRAD needs TMA-fed operands");
        }
        p.SH = g.h; p.SW = g.w; p.SC = g.c; p.sld = g.ldx;
        p.OH = g.p; p.OW = g.q; p.ald = g.ldy;
        p.dld = kpad;
        p.split_stride = (long long)g.k * kpad;
        if (p.wseg) {  // each member's partials [splits][64][kpad], members back to back
          p.split_stride = 64LL * kpad;
          p.dseg = (long long)p.splits * 64 * kpad;
        }
      }
      p.tiles_m = cdiv(p.M, cg::BM);
      p.tiles_n = cdiv(p.N, ntile);
      p.tile0 = tiles;
      tiles += p.tiles_m * p.tiles_n * p.splits;
    }
    L.total_tiles = tiles;
    // halo tiles (k_conv_gemm_halo): every problem a 3x3 stride-1 pad-1 FPROP / DGRAD on
    // a TMA-fed plane with C % 64 == 0 and >= 14-wide rows
    {
      pk_plan_options po;
      pk_plan_options_get(&po);
      // (measured, tools/gemm_probe.py halo: 14x14x256 N=256 tiles 46.6 -> 38.4 us; with
      // N <= 128 the one-CTA-per-SM halo kernel trails the two-CTA im2col kernel)
      // C == 64 with <= 64-wide N tiles: the weights-resident form (k_conv_gemm_halo_res)
      bool halo = po.conv_halo && kind != PK_CNN_CONV_WGRAD && (ntile == 256 || ntile <= 64);
      bool res = ntile <= 64;
      int maxab = 0;
      for (int j = 0; j < L.nprob && halo; ++j) {
        const cg::Problem& p = L.p[j];
        const int pw = p.OW + 2, hrows = 4 + cg::BM / pw;
        halo = p.a_mode == 2 && p.R == 3 && p.S == 3 && p.stride == 1 && p.pad == 1 &&
               p.SC % 64 == 0 && p.OW >= 14 && pw <= 256 && p.OH == p.SH && p.OW == p.SW &&
               hrows * pw * 128 <= 64 * 1024;
        maxab = std::max(maxab, rup(hrows * pw * 128, 1024));
        res = res && p.SC == 64 && p.tiles_n == 1;
      }
      if (halo && ntile <= 64 && !res) halo = false;
      if (halo) {
        tiles = 0;
        for (int j = 0; j < L.nprob; ++j) {
          const pk_cnn_conv& g = pr[i0 + j];
          cg::Problem& p = L.p[j];
          p.pw = p.OW + 2;
          p.hrows = 4 + cg::BM / p.pw;
          p.tpi = cdiv((long long)p.OH * p.pw, cg::BM);
          p.tiles_m = g.n * p.tpi;
          p.tile0 = tiles;
          tiles += p.tiles_m * p.tiles_n;
          // the input plane as a tiled 4-D map {C, W, H, N}, box {64, W + 2, hrows, 1}
          cuuint64_t dims[4] = {(cuuint64_t)p.SC, (cuuint64_t)p.SW, (cuuint64_t)p.SH,
                                (cuuint64_t)g.n};
          cuuint64_t strides[3] = {(cuuint64_t)p.sld * 2, (cuuint64_t)p.SW * p.sld * 2,
                                   (cuuint64_t)p.SH * p.SW * p.sld * 2};
          cuuint32_t box[4] = {64, (cuuint32_t)p.pw, (cuuint32_t)p.hrows, 1};
          cuuint32_t es[4] = {1, 1, 1, 1};
          if (!encode_fn() ||
              g_encode(&L.tmA[j], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(
                           static_cast<const void*>(p.src)), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return fail(PK_ERR_CUDA, "conv: halo tensor map");
        }
        L.total_tiles = tiles;
        L.halo = res ? 2 : 1;
        L.abytes = maxab;
        static int sms_h = 0;
        if (!sms_h) cudaDeviceGetAttribute(&sms_h, cudaDevAttrMultiProcessorCount, 0);
        const size_t room = (size_t)(227 * 1024) - 2 * (size_t)maxab - 4096;
        L.stages = (int)std::min<size_t>(8, room / ((size_t)ntile * 128));
        L.persistent = 1;
        L.grid = std::min(tiles, std::max(sms_h, 1));
        out.push_back(L);
        continue;
      }
    }
    // persistent when every problem's operands come by TMA (the epilogue warps are free)
    bool all_tma = true;
    for (int j = 0; j < L.nprob; ++j)
      all_tma = all_tma && (kind == PK_CNN_CONV_WGRAD ? L.p[j].b_mode != 0 : L.p[j].a_mode != 0);
    if (all_tma && tiles > 0) {
      static int sms = 0;
      if (!sms) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
      const int per_sm = 2 * ntile <= 256 ? 2 : 1;  // TMEM: 2 x NT columns per CTA
      const size_t budget = (size_t)(227 * 1024) / per_sm - 2048;
      L.stages = (int)std::min<size_t>(8, budget / cg::stage_bytes(ntile));
      L.persistent = 1;
      L.grid = std::min(tiles, per_sm * std::max(sms, 1));
      // CTA pairs sharing the weight tile (k_conv_gemm_pc): FPROP / DGRAD whose
      // activations come by 2-D / im2col TMA maps; the weight maps are re-encoded
      // with half-height boxes (each CTA of a pair loads and multicasts one half)
      pk_plan_options po;
      pk_plan_options_get(&po);
      bool pair = po.conv_cluster && kind != PK_CNN_CONV_WGRAD && ntile % 32 == 0;
      // (short-K GEMMs — 1x1 convs with K < 512 — are epilogue-bound: no gain, measured)
      for (int j = 0; j < L.nprob && pair; ++j)
        pair = (L.p[j].a_mode == 1 || L.p[j].a_mode == 2) && L.p[j].splits == 1 &&
               L.p[j].K >= 512 && L.p[j].par < 0;
      if (pair) {
        int pairs = 0;
        for (int j = 0; j < L.nprob; ++j) {
          const pk_cnn_conv& g = pr[i0 + j];
          cg::Problem& p = L.p[j];
          const bool ok =
              kind == PK_CNN_CONV_FPROP
                  ? make_map_2d(&L.tm[j], g.wt, g.k, rup(g.r * g.s * g.c, 64),
                                rup(g.r * g.s * g.c, 64), ntile / 2)
                  : make_map_2d(&L.tm[j], g.wt, g.c, rup(g.r * g.s * g.k, 64),
                                rup(g.r * g.s * g.k, 64), ntile / 2);
          if (!ok) return fail(PK_ERR_CUDA, "conv: half-box weight map");
          p.pair0 = pairs;
          pairs += (p.tiles_m + 1) / 2 * p.tiles_n;
        }
        L.cluster = 2;
        L.total_pairs = pairs;
        L.grid = 2 * std::min(pairs, std::max(1, per_sm * std::max(sms, 1) / 2));
        if (po.conv_cluster == 2 && (ntile == 64 || ntile == 128 || ntile == 256)) {
          // CTA-pair MMA: half of B per CTA → deeper rings in the same smem
          L.pair_mma = 1;
          const int ps = ntile == 256 ? 1 : 2;  // TMEM: 2 x NT columns per CTA
          const size_t budget2 = (size_t)(227 * 1024) / ps - 2048;
          L.stages = (int)std::min<size_t>(8, budget2 / cg::stage_bytes_pair(ntile));
          L.grid = 2 * std::min(pairs, std::max(1, ps * std::max(sms, 1) / 2));
        }
      }
    }
    out.push_back(L);
  }
  return PK_OK;
}

// Every launch of a step program after its first carries the programmatic-
// stream-serialization attribute (PDL): the kernels open with pdl_gate(), so the
// next launch is placed while the current one drains.  t_pdl is cleared at the
// start of a program (its first launch follows unrelated stream work) and by the
// per-op profiler / the single-GEMM test entry (events between launches).
thread_local bool t_pdl = false;

template <class... KArgs, class... Args>
cudaError_t launch_kx(void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t st,
                      int cluster, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (t_pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (cluster > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = (unsigned)cluster;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  t_pdl = true;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
template <class... KArgs, class... Args>
cudaError_t launch_k(void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t st,
                     Args&&... args) {
  return launch_kx(kern, grid, block, smem, st, 1, std::forward<Args>(args)...);
}

template <int MODE>
cudaError_t launch_conv(const cg::Launch& L, cudaStream_t st) {
  static bool attr_set = false, attr_set_p = false, attr_set_c = false;
  if (L.total_tiles == 0) return cudaSuccess;
  if (L.halo == 2) {
    if constexpr (MODE != cg::WGRAD) {
      static bool attr_set_r = false;
      if (!attr_set_r) {
        cudaError_t e = cudaFuncSetAttribute(cg::k_conv_gemm_halo_res<MODE>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             227 * 1024);
        if (e != cudaSuccess) return e;
        attr_set_r = true;
      }
      const size_t smr = 1024 + 2 * (size_t)L.abytes + 9 * (size_t)L.ntile * 128 + 8 * 10 + 16;
      return launch_k(cg::k_conv_gemm_halo_res<MODE>, L.grid, cg::kThreads, smr, st, L);
    }
    return cudaErrorInvalidValue;
  }
  if (L.halo) {
    if constexpr (MODE != cg::WGRAD) {
      static bool attr_set_h = false;
      if (!attr_set_h) {
        cudaError_t e = cudaFuncSetAttribute(cg::k_conv_gemm_halo<MODE>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             227 * 1024);
        if (e != cudaSuccess) return e;
        attr_set_h = true;
      }
      const size_t smh = 1024 + 2 * (size_t)L.abytes + (size_t)L.stages * L.ntile * 128 +
                         8 * (2 * L.stages + 8) + 16;
      return launch_k(cg::k_conv_gemm_halo<MODE>, L.grid, cg::kThreads, smh, st, L);
    }
    return cudaErrorInvalidValue;
  }
  if (L.cluster == 2 && L.pair_mma) {
    if constexpr (MODE != cg::WGRAD) {
      static bool attr_set_2 = false;
      if (!attr_set_2) {
        cudaError_t e = cudaFuncSetAttribute(cg::k_conv_gemm_p2<MODE>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             227 * 1024);
        if (e != cudaSuccess) return e;
        attr_set_2 = true;
      }
      const size_t sm2 = 1024 + (size_t)L.stages * cg::stage_bytes_pair(L.ntile) +
                         8 * (2 * L.stages + 4) + 16;
      return launch_kx(cg::k_conv_gemm_p2<MODE>, L.grid, cg::kThreads, sm2, st, 2, L);
    }
    return cudaErrorInvalidValue;
  }
  if (L.cluster == 2) {
    if constexpr (MODE != cg::WGRAD) {
      if (!attr_set_c) {
        cudaError_t e = cudaFuncSetAttribute(cg::k_conv_gemm_pc<MODE>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             227 * 1024);
        if (e != cudaSuccess) return e;
        attr_set_c = true;
      }
      return launch_kx(cg::k_conv_gemm_pc<MODE>, L.grid, cg::kThreads,
                       cg::smem_bytes(L.ntile, L.stages), st, 2, L);
    }
    return cudaErrorInvalidValue;
  }
  if (L.persistent) {
    if (!attr_set_p) {
      cudaError_t e = cudaFuncSetAttribute(cg::k_conv_gemm_p<MODE>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      if (e != cudaSuccess) return e;
      attr_set_p = true;
    }
    return launch_k(cg::k_conv_gemm_p<MODE>, L.grid, cg::kThreads,
                    cg::smem_bytes(L.ntile, L.stages), st, L);
  }
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(cg::k_conv_gemm<MODE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  return launch_k(cg::k_conv_gemm<MODE>, L.total_tiles, cg::kThreads,
                  cg::smem_bytes(L.ntile, L.stages), st, L);
}

template <class P>
const P* dp(const pk_cnn_prog* g, const OpRec& o) {
  return reinterpret_cast<const P*>(g->dmem + o.probs_off);
}
const int* db(const pk_cnn_prog* g, const OpRec& o) {
  return reinterpret_cast<const int*>(g->dmem + o.blk_off);
}

template <class T>
cudaError_t launch_packs(const OpRec& o, void (*kern)(cnn::Pack<T>), cudaStream_t st,
                         int smem = 0) {
  for (size_t i = 0; i < o.packs.size(); ++i) {
    if (o.pack_blocks[i] == 0) continue;
    cudaError_t e = launch_k(kern, o.pack_blocks[i], cnn::kBlock, smem, st,
                             *reinterpret_cast<const cnn::Pack<T>*>(o.packs[i].data()));
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t run_op(const pk_cnn_prog* g, const OpRec& o, cudaStream_t st) {
  using namespace cnn;
  const int nb = o.nblocks, np = o.nprob;
  switch (o.kind) {
    case PK_CNN_CONV_FPROP:
      for (auto& L : o.conv) {
        cudaError_t e = launch_conv<cg::FPROP>(L, st);
        if (e != cudaSuccess) return e;
      }
      return cudaSuccess;
    case PK_CNN_CONV_DGRAD:
      for (auto& L : o.conv) {
        cudaError_t e = launch_conv<cg::DGRAD>(L, st);
        if (e != cudaSuccess) return e;
      }
      return cudaSuccess;
    case PK_CNN_CONV_WGRAD:
      for (auto& L : o.conv) {
        cudaError_t e = launch_conv<cg::WGRAD>(L, st);
        if (e != cudaSuccess) return e;
      }
      return cudaSuccess;
    case PK_CNN_BN_STATS: return launch_packs<pk_cnn_bn>(o, k_bn_stats, st);
    case PK_CNN_BN_APPLY: return launch_packs<pk_cnn_bn>(o, k_bn_apply, st);
    case PK_CNN_BN_BWD_REDUCE: return launch_packs<pk_cnn_bn>(o, k_bn_bwd_reduce, st);
    case PK_CNN_BN_BWD_APPLY:
      for (size_t i = 0; i < o.packs.size(); ++i) {  // variant per pack: activation, side outputs
        if (o.pack_blocks[i] == 0) continue;
        const auto& P = *reinterpret_cast<const cnn::Pack<pk_cnn_bn>*>(o.packs[i].data());
        bool act = false, side = false;
        for (int j = 0; j < P.nprob; ++j) {
          act = act || P.p[j].act != PK_CNN_ACT_NONE;
          side = side || P.p[j].accumulate || P.p[j].dres;
        }
        auto kern = act ? (side ? k_bn_bwd_apply_t<true, true> : k_bn_bwd_apply_t<true, false>)
                        : (side ? k_bn_bwd_apply_t<false, true> : k_bn_bwd_apply_t<false, false>);
        cudaError_t e = launch_k(kern, o.pack_blocks[i], kBlock, 0, st, P);
        if (e != cudaSuccess) return e;
      }
      return cudaSuccess;
    case PK_CNN_DW_FPROP: return launch_packs<pk_cnn_dw>(o, k_dw_fprop, st);
    case PK_CNN_DW_DGRAD: return launch_packs<pk_cnn_dw>(o, k_dw_dgrad, st);
    case PK_CNN_DW_WGRAD: return launch_packs<pk_cnn_dw>(o, k_dw_wgrad, st);
    case PK_CNN_MAXPOOL_FWD: return launch_packs<pk_cnn_pool>(o, k_maxpool_fwd, st);
    case PK_CNN_MAXPOOL_BWD: return launch_packs<pk_cnn_pool>(o, k_maxpool_bwd, st);
    case PK_CNN_AVGPOOL_FWD: return launch_packs<pk_cnn_pool>(o, k_avgpool_fwd, st);
    case PK_CNN_AVGPOOL_BWD: return launch_packs<pk_cnn_pool>(o, k_avgpool_bwd, st);
    case PK_CNN_XENT: return launch_packs<pk_cnn_head>(o, k_xent, st, o.ntile);
    case PK_CNN_BIAS_ACT_BWD: return launch_packs<pk_cnn_bias>(o, k_bias_act_bwd, st);
    case PK_CNN_SPLIT_REDUCE: return launch_packs<pk_cnn_reduce>(o, k_split_reduce, st);
    case PK_CNN_OPT: return launch_k(k_opt, nb, kBlock, 0, st, dp<pk_cnn_opt_seg>(g, o), db(g, o), np);
    case PK_CNN_PUBLISH_T: return launch_packs<pk_cnn_tpose>(o, k_publish_t, st);
    case PK_CNN_GATHER: return launch_packs<pk_cnn_gather>(o, k_gather, st);
    case PK_CNN_IM2COL: return launch_packs<pk_cnn_im2col>(o, k_im2col, st);
    case PK_CNN_COMMIT:
      return launch_k(k_commit, cdiv(np, 128), 128, 0, st, dp<pk_cnn_commit>(g, o), np, o.ntile);
  }
  return cudaGetLastError();
}

// Lanes: lane-0 ops run on `st`; a lane L > 0 forks from `st` (event) at its
// first op after a lane-0 op and joins `st` (event) before the next lane-0 op.
// PDL chains each lane's launches; the first launch after a fork or a join
// carries no PDL attribute (its predecessor is an event, not a kernel).
int run_all(pk_cnn_prog* g, cudaStream_t st) {
  bool pdl[kMaxLanes + 1] = {}, open[kMaxLanes + 1] = {}, aopen[kMaxLanes + 1] = {};
  bool any_open = false, forked = false, any_async = false;
  // async lanes join the program stream before the commit / optimizer ops (and at the end)
  auto join_async = [&]() -> cudaError_t {
    cudaError_t e = cudaSuccess;
    for (int a = 1; a <= kMaxLanes && e == cudaSuccess; ++a)
      if (aopen[a]) {
        e = cudaEventRecord(g->async_join[a], g->async_st[a]);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, g->async_join[a], 0);
        aopen[a] = false;
      }
    any_async = false;
    pdl[0] = false;
    return e;
  };
  for (size_t i = 0; i < g->ops.size(); ++i) {
    const int L = g->ops[i].lane;
    cudaError_t e = cudaSuccess;
    if (L >= 16) {  // async op: waits for everything the program stream has issued so far
      const int a = L - 16;
      if (!g->async_st[a]) {
        e = cudaStreamCreateWithFlags(&g->async_st[a], cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g->async_fork[a], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g->async_join[a], cudaEventDisableTiming);
      }
      // parent: the sync lane a while it is open (heterogeneous packs), else the program
      // stream
      cudaStream_t parent = open[a] ? g->lane_st[a] : st;
      if (e == cudaSuccess) e = cudaEventRecord(g->async_fork[a], parent);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(g->async_st[a], g->async_fork[a], 0);
      if (e == cudaSuccess) {
        t_pdl = false;
        e = run_op(g, g->ops[i], g->async_st[a]);
      }
      aopen[a] = any_async = true;
      if (e != cudaSuccess)
        return fail(PK_ERR_CUDA, "op " + std::to_string(i) + " (async): " + cudaGetErrorString(e));
      continue;
    }
    if (any_async && (g->ops[i].kind == PK_CNN_COMMIT || g->ops[i].kind == PK_CNN_OPT))
      e = join_async();
    if (e == cudaSuccess && L == 0 && any_open) {  // join every lane opened since the last lane-0 op
      for (int l = 1; l <= kMaxLanes && e == cudaSuccess; ++l)
        if (open[l]) {
          e = cudaEventRecord(g->join_ev[l], g->lane_st[l]);
          if (e == cudaSuccess) e = cudaStreamWaitEvent(st, g->join_ev[l], 0);
          open[l] = false;
        }
      any_open = forked = false;
      pdl[0] = false;
    } else if (L > 0 && !open[L]) {
      if (!g->lane_st[L]) {
        e = cudaStreamCreateWithFlags(&g->lane_st[L], cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g->join_ev[L], cudaEventDisableTiming);
        if (e == cudaSuccess && !g->fork_ev)
          e = cudaEventCreateWithFlags(&g->fork_ev, cudaEventDisableTiming);
      }
      if (e == cudaSuccess && !forked) {
        e = cudaEventRecord(g->fork_ev, st);
        forked = true;
      }
      if (e == cudaSuccess) e = cudaStreamWaitEvent(g->lane_st[L], g->fork_ev, 0);
      open[L] = any_open = true;
      pdl[L] = false;
    }
    if (e == cudaSuccess) {
      t_pdl = pdl[L];
      e = run_op(g, g->ops[i], L ? g->lane_st[L] : st);
      pdl[L] = t_pdl;
    }
    if (e != cudaSuccess)
      return fail(PK_ERR_CUDA, "op " + std::to_string(i) + " (kind " +
                                   std::to_string(g->ops[i].kind) + "): " + cudaGetErrorString(e));
  }
  if (any_open) {  // a program ending in lane ops still joins
    for (int l = 1; l <= kMaxLanes; ++l)
      if (open[l]) {
        cudaError_t e = cudaEventRecord(g->join_ev[l], g->lane_st[l]);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, g->join_ev[l], 0);
        if (e != cudaSuccess) return fail(PK_ERR_CUDA, cudaGetErrorString(e));
      }
  }
  if (any_async) {
    cudaError_t e = join_async();
    if (e != cudaSuccess) return fail(PK_ERR_CUDA, cudaGetErrorString(e));
  }
  return PK_OK;
}

}  // namespace

extern "C" const char* pk_cnn_last_error(void) { return g_err.c_str(); }

extern "C" int pk_cnn_prog_create(const pk_cnn_op* ops, int32_t nops, int32_t device,
                                  pk_cnn_prog** out) {
  if (!ops || nops <= 0 || !out) return fail(PK_ERR_ARG, "pk_cnn_prog_create: no ops");
  *out = nullptr;
  if (cudaSetDevice(device) != cudaSuccess) return fail(PK_ERR_CUDA, "cudaSetDevice failed");
  auto* g = new pk_cnn_prog();
  g->device = device;
  std::vector<uint8_t> host;
  auto align = [&](size_t a) { host.resize((host.size() + a - 1) / a * a); };
  for (int i = 0; i < nops; ++i) {
    const pk_cnn_op& op = ops[i];
    OpRec r;
    r.kind = op.kind;
    r.nprob = op.nprob;
    r.lane = op.lane;
    if (op.lane < 0 || (op.lane > kMaxLanes && (op.lane < 17 || op.lane > 16 + kMaxLanes))) {
      delete g;
      return fail(PK_ERR_ARG, "op " + std::to_string(i) + ": lane out of range");
    }
    const size_t ps = prob_size(op.kind);
    if (!ps || op.nprob <= 0 || !op.probs) {
      delete g;
      return fail(PK_ERR_ARG, "op " + std::to_string(i) + ": bad kind or no problems");
    }
    if (op.kind <= PK_CNN_CONV_WGRAD) {
      r.ntile = op.cfg0;
      r.stages = op.cfg1;
      if (r.ntile < 16 || r.ntile > 256 || r.ntile % 16 || r.stages < 2 ||
          cg::smem_bytes(r.ntile, r.stages) > 227 * 1024) {
        delete g;
        return fail(PK_ERR_ARG, "op " + std::to_string(i) + ": bad conv tile / stages");
      }
      int rc = conv_to_launches(op.kind, static_cast<const pk_cnn_conv*>(op.probs), op.nprob,
                                r.ntile, r.stages, r.conv);
      if (rc != PK_OK) {
        delete g;
        return rc;
      }
      g->launches += (int)r.conv.size();
      g->ops.push_back(std::move(r));
      continue;
    }
    std::vector<int> blk(op.nprob + 1, 0);
    const uint8_t* src = static_cast<const uint8_t*>(op.probs);
    for (int j = 0; j < op.nprob; ++j) {
      std::string why = check_prob(op.kind, src + j * ps);
      if (!why.empty()) {
        delete g;
        return fail(PK_ERR_ARG, "op " + std::to_string(i) + ": " + why);
      }
      blk[j + 1] = blk[j] + prob_blocks(op.kind, src + j * ps);
    }
    r.nblocks = blk[op.nprob];
    if (op.kind == PK_CNN_COMMIT) r.ntile = op.cfg0;  // mode
    if (op.kind != PK_CNN_OPT && op.kind != PK_CNN_COMMIT) {
      if (op.kind == PK_CNN_XENT) {
        int mx = 0;
        for (int j = 0; j < op.nprob; ++j)
          mx = std::max(mx, reinterpret_cast<const pk_cnn_head*>(src)[j].rows);
        r.ntile = mx * 16 + cdiv(mx, 32) * 32 * 4;  // dynamic smem bytes (k_xent layout)
      }
      switch (op.kind) {
        case PK_CNN_BN_STATS:
        case PK_CNN_BN_APPLY:
        case PK_CNN_BN_BWD_REDUCE:
        case PK_CNN_BN_BWD_APPLY:
          make_packs(r, static_cast<const pk_cnn_bn*>(op.probs), op.nprob, prob_blocks);
          break;
        case PK_CNN_DW_FPROP:
        case PK_CNN_DW_DGRAD:
        case PK_CNN_DW_WGRAD:
          make_packs(r, static_cast<const pk_cnn_dw*>(op.probs), op.nprob, prob_blocks);
          break;
        case PK_CNN_MAXPOOL_FWD:
        case PK_CNN_MAXPOOL_BWD:
        case PK_CNN_AVGPOOL_FWD:
        case PK_CNN_AVGPOOL_BWD:
          make_packs(r, static_cast<const pk_cnn_pool*>(op.probs), op.nprob, prob_blocks);
          break;
        case PK_CNN_XENT:
          make_packs(r, static_cast<const pk_cnn_head*>(op.probs), op.nprob, head_blocks);
          break;
        case PK_CNN_BIAS_ACT_BWD:
          make_packs(r, static_cast<const pk_cnn_bias*>(op.probs), op.nprob, prob_blocks);
          break;
        case PK_CNN_SPLIT_REDUCE:
          make_packs(r, static_cast<const pk_cnn_reduce*>(op.probs), op.nprob, prob_blocks);
          break;
        case PK_CNN_PUBLISH_T:
          make_packs(r, static_cast<const pk_cnn_tpose*>(op.probs), op.nprob, prob_blocks);
          break;
        case PK_CNN_GATHER:
          make_packs(r, static_cast<const pk_cnn_gather*>(op.probs), op.nprob, prob_blocks);
          break;
        case PK_CNN_IM2COL:
          make_packs(r, static_cast<const pk_cnn_im2col*>(op.probs), op.nprob, prob_blocks);
          break;
      }
      g->launches += (int)r.packs.size();
      g->ops.push_back(std::move(r));
      continue;
    }
    align(64);
    r.probs_off = host.size();
    host.insert(host.end(), src, src + ps * op.nprob);
    align(16);
    r.blk_off = host.size();
    const uint8_t* b = reinterpret_cast<const uint8_t*>(blk.data());
    host.insert(host.end(), b, b + sizeof(int) * blk.size());
    g->launches += 1;
    g->ops.push_back(std::move(r));
  }
  if (!host.empty()) {
    if (cudaMalloc(&g->dmem, host.size()) != cudaSuccess) {
      delete g;
      return fail(PK_ERR_OOM, "pk_cnn_prog_create: descriptor allocation failed");
    }
    if (cudaMemcpy(g->dmem, host.data(), host.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
      cudaFree(g->dmem);
      delete g;
      return fail(PK_ERR_CUDA, "pk_cnn_prog_create: descriptor upload failed");
    }
  }
  *out = g;
  return PK_OK;
}

extern "C" void pk_cnn_prog_destroy(pk_cnn_prog* g) {
  if (!g) return;
  if (g->gexec) cudaGraphExecDestroy(g->gexec);
  for (int l = 1; l <= kMaxLanes; ++l) {
    if (g->lane_st[l]) cudaStreamDestroy(g->lane_st[l]);
    if (g->join_ev[l]) cudaEventDestroy(g->join_ev[l]);
    if (g->async_st[l]) cudaStreamDestroy(g->async_st[l]);
    if (g->async_fork[l]) cudaEventDestroy(g->async_fork[l]);
    if (g->async_join[l]) cudaEventDestroy(g->async_join[l]);
  }
  if (g->fork_ev) cudaEventDestroy(g->fork_ev);
  if (g->dmem) cudaFree(g->dmem);
  delete g;
}

extern "C" int32_t pk_cnn_prog_launches(const pk_cnn_prog* g) { return g ? g->launches : 0; }

extern "C" int pk_cnn_prog_run(pk_cnn_prog* g, void* stream, int32_t use_graph) {
  if (!g) return fail(PK_ERR_ARG, "pk_cnn_prog_run: null program");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!use_graph) return run_all(g, st);
  if (!g->gexec) {
    cudaGraph_t graph = nullptr;
    if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
      return fail(PK_ERR_CUDA, "pk_cnn_prog_run: cannot capture on this stream (legacy default "
                               "stream?)");
    int rc = run_all(g, st);
    cudaError_t e = cudaStreamEndCapture(st, &graph);
    if (rc != PK_OK) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    if (e != cudaSuccess) return fail(PK_ERR_CUDA, std::string("capture: ") + cudaGetErrorString(e));
    e = cudaGraphInstantiate(&g->gexec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
      g->gexec = nullptr;
      return fail(PK_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    }
  }
  cudaError_t e = cudaGraphLaunch(g->gexec, st);
  return e == cudaSuccess ? PK_OK : fail(PK_ERR_CUDA, cudaGetErrorString(e));
}

extern "C" int pk_cnn_prog_profile(pk_cnn_prog* g, void* stream, float* op_ms) {
  if (!g || !op_ms) return fail(PK_ERR_ARG, "pk_cnn_prog_profile: null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t n = g->ops.size();
  // events around every op; a ~40 µs device spin ahead of each op keeps the GPU
  // busy while the host enqueues the op, so an op's time is its own device time
  // (its kernels' launch on the GPU included), not the host's enqueue latency
  std::vector<cudaEvent_t> ev(2 * n);
  for (auto& e : ev) cudaEventCreate(&e);
  int rc = PK_OK;
  for (size_t i = 0; i < n && rc == PK_OK; ++i) {
    cnn::k_spin<<<1, 32, 0, st>>>(80000);
    cudaEventRecord(ev[2 * i], st);
    t_pdl = false;
    cudaError_t e = run_op(g, g->ops[i], st);
    if (e != cudaSuccess) rc = fail(PK_ERR_CUDA, cudaGetErrorString(e));
    cudaEventRecord(ev[2 * i + 1], st);
  }
  if (n && cudaEventSynchronize(ev[2 * n - 1]) != cudaSuccess && rc == PK_OK)
    rc = fail(PK_ERR_CUDA, "pk_cnn_prog_profile: synchronize failed");
  for (size_t i = 0; i < n && rc == PK_OK; ++i)
    cudaEventElapsedTime(&op_ms[i], ev[2 * i], ev[2 * i + 1]);
  for (auto& e : ev) cudaEventDestroy(e);
  return rc;
}

extern "C" int pk_conv_gemm_test(int32_t mode, const pk_conv_geom* g, const void* x,
                                 const void* w, const void* dy, void* out, int32_t ntile,
                                 int32_t splits, int32_t stages, void* stream) {
  if (!g || mode < 0 || mode > 2 || ntile < 16 || ntile > 256 || ntile % 16 || stages < 2 ||
      stages > 6 || g->c % 8 || g->k % 8 || (g->stride != 1 && g->stride != 2))
    return PK_ERR_ARG;
  if (mode == 2 && ntile % 64) return PK_ERR_ARG;
  static cg::Launch L;
  memset(&L, 0, sizeof(L));
  L.nprob = 1;
  L.p[0].par = -1;
  L.ntile = ntile;
  L.stages = stages;
  cg::Problem& p = L.p[0];
  p.R = g->r;
  p.S = g->s;
  p.stride = g->stride;
  p.pad = g->pad;
  CUtensorMap& tm = L.tm[0];
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaSuccess;
  if (mode == 0) {
    const int kpad = rup(g->r * g->s * g->c, 64);
    p.src = static_cast<const __nv_bfloat16*>(x);
    p.dst = out;
    p.M = g->n * g->p * g->q;
    p.N = g->k;
    p.K = g->r * g->s * g->c;
    p.SH = g->h; p.SW = g->w; p.SC = g->c; p.sld = g->c;
    p.OH = g->p; p.OW = g->q;
    p.dld = g->k;
    if (!make_map_2d(&tm, w, g->k, kpad, kpad, ntile)) return PK_ERR_CUDA;
    e = launch_gemm<cg::FPROP>(L, st);
  } else if (mode == 1) {
    const int kpad = rup(g->r * g->s * g->k, 64);
    p.src = static_cast<const __nv_bfloat16*>(dy);
    p.dst = out;
    p.M = g->n * g->h * g->w;
    p.N = g->c;
    p.K = g->r * g->s * g->k;
    p.SH = g->p; p.SW = g->q; p.SC = g->k; p.sld = g->k;
    p.OH = g->h; p.OW = g->w;
    p.dld = g->c;
    if (!make_map_2d(&tm, w, g->c, kpad, kpad, ntile)) return PK_ERR_CUDA;
    e = launch_gemm<cg::DGRAD>(L, st);
  } else {
    const int kpad = rup(g->r * g->s * g->c, 64);
    const int pix = g->n * g->p * g->q;
    p.src = static_cast<const __nv_bfloat16*>(x);
    p.src2 = static_cast<const __nv_bfloat16*>(dy);
    p.dst = out;
    p.M = g->k;
    p.N = g->r * g->s * g->c;
    p.K = pix;
    p.splits = std::max(1, splits);
    p.kper = rup(cdiv(pix, p.splits), 64);
    p.splits = cdiv(pix, p.kper);
    p.SH = g->h; p.SW = g->w; p.SC = g->c; p.sld = g->c;
    p.OH = g->p; p.OW = g->q;
    p.ald = g->k;
    p.dld = kpad;
    p.split_stride = (long long)g->k * kpad;
    e = launch_gemm<cg::WGRAD>(L, st);
  }
  return e == cudaSuccess ? PK_OK : PK_ERR_CUDA;
}
