// pk_cnn.cu — conv pack runtime behind the packtrain_b200.h C-ABI (pk_cnet_*).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
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

// 2-D bf16 tensor map [rows][cols] (row pitch `ld` elements), box {64, box_rows}, SW128
bool make_map_2d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                 uint32_t box_rows) {
  if (!encode_fn()) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  return g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }
inline int rup(int a, int b) { return (a + b - 1) / b * b; }

// fill tile counts / prefix and launch one grouped implicit-GEMM conv
template <int MODE>
cudaError_t launch_gemm(cg::Launch& L, const CUtensorMap& tm, cudaStream_t st) {
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
  cg::k_conv_gemm<MODE><<<tiles, cg::kThreads, smem, st>>>(L, tm);
  return cudaGetLastError();
}

}  // namespace

extern "C" int pk_conv_gemm_test(int32_t mode, const pk_conv_geom* g, const void* x,
                                 const void* w, const void* dy, void* out, int32_t ntile,
                                 int32_t splits, int32_t stages, void* stream) {
  if (!g || mode < 0 || mode > 2 || ntile < 16 || ntile > 256 || ntile % 16 || stages < 2 ||
      stages > 6 || g->c % 8 || g->k % 8 || (g->stride != 1 && g->stride != 2))
    return PK_ERR_ARG;
  if (mode == 2 && ntile % 64) return PK_ERR_ARG;
  cg::Launch L;
  memset(&L, 0, sizeof(L));
  L.nprob = 1;
  L.ntile = ntile;
  L.stages = stages;
  cg::Problem& p = L.p[0];
  p.R = g->r;
  p.S = g->s;
  p.stride = g->stride;
  p.pad = g->pad;
  CUtensorMap tm;
  memset(&tm, 0, sizeof(tm));
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
    e = launch_gemm<cg::FPROP>(L, tm, st);
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
    e = launch_gemm<cg::DGRAD>(L, tm, st);
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
    e = launch_gemm<cg::WGRAD>(L, tm, st);
  }
  return e == cudaSuccess ? PK_OK : PK_ERR_CUDA;
}
