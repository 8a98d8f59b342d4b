// pk_runtime.cu — host runtime behind the packtrain_b200.h C-ABI.
//
// Owns device memory (datasets, epoch orders, member slabs), builds the
// per-pack tile schedule, captures the step's kernel sequence in a CUDA graph
// and drives it: one H2D copy of the step descriptor + one graph launch per
// packed step; the finalize kernel writes {status, losses} straight into a
// host-mapped ring, so the host sync is the only per-step round trip.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstddef>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "packtrain_b200.h"
#include "pk_kernels.cuh"

using pk::FeedDev;
using pk::MemberCtl;
using pk::MemberDev;
using pk::StepHdr;
using pk::Tile;

namespace {
constexpr int kRing = 32;  // in-flight step descriptors / result slots
size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }
}  // namespace

struct pk_ctx {
  int device = 0;
  int dtype = PK_F32;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::string err;
  uint64_t bytes = 0;
  size_t esize() const { return dtype == PK_F64 ? 8 : 4; }
  // recycled per-pack buffers and events: Hyperband builds and drops a pack
  // per group evaluation, and cudaFree / cudaFreeHost / cudaHostAlloc cost
  // milliseconds each (kind 0 device, 1 pinned, 2 pinned + mapped)
  struct Block {
    void* p;
    size_t cap;
    int kind;
  };
  std::vector<Block> blocks;
  // device blocks up to kArenaBlock are carved from 64 MiB arenas: a cache
  // miss costs no cudaMalloc (Hyperband creates a member slab per new
  // configuration); arena blocks stay cached until the context is destroyed
  std::vector<std::pair<char*, size_t>> arenas;
  char* arena_cur = nullptr;
  size_t arena_left = 0;
  std::vector<cudaEvent_t> events;
};

static const char* const kAllocKind[] = {"device", "pinned", "mapped"};
constexpr size_t kArenaBlock = size_t(8) << 20, kArenaBytes = size_t(64) << 20;
// arenas are never returned while the context lives (their blocks are recycled
// through the block cache); past this many, small blocks get their own
// cudaMalloc and fall under the cache's entry / byte bound like large ones
constexpr size_t kMaxArenas = 16;

// a cached block of `kind` with bytes <= cap <= slack·bytes, else a fresh one
static cudaError_t ctx_alloc(pk_ctx* c, int kind, size_t bytes, void** out, size_t* cap,
                             double slack = 4.0) {
  bytes = std::max<size_t>(bytes, 256);
  size_t best = SIZE_MAX, bi = 0;
  for (size_t i = 0; i < c->blocks.size(); ++i) {
    const auto& b = c->blocks[i];
    if (b.kind == kind && b.cap >= bytes && (double)b.cap <= slack * (double)bytes && b.cap < best) {
      best = b.cap;
      bi = i;
    }
  }
  if (best != SIZE_MAX) {
    *out = c->blocks[bi].p;
    *cap = best;
    c->blocks.erase(c->blocks.begin() + bi);
    return cudaSuccess;
  }
  *cap = bytes;
  const size_t need = (bytes + 255) & ~size_t(255);
  if (kind == 0 && bytes <= kArenaBlock &&
      (c->arena_left >= need || c->arenas.size() < kMaxArenas)) {
    if (c->arena_left < need) {
      char* a = nullptr;
      cudaError_t e = cudaMalloc(&a, kArenaBytes);
      if (e != cudaSuccess) return e;
      c->arenas.push_back({a, kArenaBytes});
      c->arena_cur = a;
      c->arena_left = kArenaBytes;
    }
    *out = c->arena_cur;
    *cap = need;
    c->arena_cur += need;
    c->arena_left -= need;
    return cudaSuccess;
  }
  if (kind == 0) return cudaMalloc(out, bytes);
  return cudaHostAlloc(out, bytes, kind == 1 ? cudaHostAllocDefault : cudaHostAllocMapped);
}

static bool ctx_in_arena(const pk_ctx* c, const void* p) {
  const char* q = static_cast<const char*>(p);
  for (const auto& a : c->arenas)
    if (q >= a.first && q < a.first + a.second) return true;
  return false;
}

static void ctx_free_block(const pk_ctx* c, const pk_ctx::Block& b) {
  if (b.kind == 0) {
    if (!ctx_in_arena(c, b.p)) cudaFree(b.p);
  } else {
    cudaFreeHost(b.p);
  }
}

static void ctx_release(pk_ctx* c, int kind, void* p, size_t cap) {
  if (!p) return;
  c->blocks.push_back({p, cap, kind});
  // bounded (entries and bytes) over the blocks that own their memory: drop
  // the oldest of those; arena blocks stay until the context goes
  size_t held = 0, owned = 0;
  for (const auto& b : c->blocks)
    if (b.kind != 0 || !ctx_in_arena(c, b.p)) held += b.cap, ++owned;
  for (size_t i = 0; i < c->blocks.size() && (owned > 512 || held > (size_t(2) << 30));) {
    const auto& b = c->blocks[i];
    if (b.kind == 0 && ctx_in_arena(c, b.p)) {
      ++i;
      continue;
    }
    held -= b.cap;
    --owned;
    ctx_free_block(c, b);
    c->blocks.erase(c->blocks.begin() + i);
  }
}

static cudaEvent_t ctx_event(pk_ctx* c) {
  if (!c->events.empty()) {
    cudaEvent_t e = c->events.back();
    c->events.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  return e;
}

struct pk_dataset {
  pk_ctx* ctx;
  int64_t n;
  int32_t dim;
  void* feat;
  int32_t* labels;
};

struct pk_order {
  pk_ctx* ctx;
  int64_t n;
  int32_t* perm;
};

struct pk_member {
  pk_ctx* ctx;
  pk_member_desc desc;
  int n_slots;
  int64_t P;
  int64_t SS;  // slot block stride: P rounded up to 16 bytes
  int64_t w_off[PK_MAX_LAYERS], b_off[PK_MAX_LAYERS];
  char* slab;
  size_t slab_bytes;
  size_t slab_cap;  // capacity of the (possibly recycled) block
  void* params[2];
  void* slots[2];
  void* Z[PK_MAX_LAYERS];
  void* A[PK_MAX_LAYERS];
  void* dZ[PK_MAX_LAYERS];
  double* rowloss;
  MemberCtl* ctl;
  bool mlp1;  // fused one-hidden-layer step
  bool m1t;   // tensor-core (tcgen05 3xTF32) one-hidden-layer step
  bool m1x;   // one-launch cluster step (pk_m1x.cuh), batch <= 64
};

struct pk_pack;

// defined in pk_pack.cuh: whether a member takes the fused one-hidden-layer
// step (pk_mlp1.cuh); decided from the member's own shape only
static bool mlp1_eligible(const pk_member_desc& d, int dtype, int device);
static bool m1t_eligible(const pk_member_desc& d, int dtype, int device);
static bool m1x_eligible(const pk_member_desc& d, int dtype, int device);

#define CK_CTX(ctx, call)                                                        \
  do {                                                                           \
    cudaError_t e_ = (call);                                                     \
    if (e_ != cudaSuccess) {                                                     \
      (ctx)->err = std::string(#call) + ": " + cudaGetErrorString(e_);           \
      return e_ == cudaErrorMemoryAllocation ? PK_ERR_OOM : PK_ERR_CUDA;         \
    }                                                                            \
  } while (0)

static int arg_err(pk_ctx* ctx, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return PK_ERR_ARG;
}

// ------------------------------------------------------------------ ctx --
extern "C" int pk_abi_version(void) { return PK_ABI_VERSION; }

extern "C" int pk_ctx_create(int32_t device, int32_t dtype, pk_ctx** out) {
  if (!out || (dtype != PK_F32 && dtype != PK_F64)) return PK_ERR_ARG;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) return PK_ERR_CUDA;
  auto* c = new pk_ctx();
  c->device = device;
  c->dtype = dtype;
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return PK_ERR_CUDA;
  }
  c->own_stream = true;
  *out = c;
  return PK_OK;
}

extern "C" int pk_ctx_destroy(pk_ctx* c) {
  if (!c) return PK_ERR_ARG;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (const auto& b : c->blocks) ctx_free_block(c, b);
  for (const auto& a : c->arenas) cudaFree(a.first);
  for (auto e : c->events) cudaEventDestroy(e);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
  return PK_OK;
}

extern "C" const char* pk_ctx_last_error(const pk_ctx* c) { return c ? c->err.c_str() : "null ctx"; }

extern "C" int pk_ctx_set_stream(pk_ctx* c, void* s) {
  if (!c) return PK_ERR_ARG;
  cudaSetDevice(c->device);
  CK_CTX(c, cudaStreamSynchronize(c->stream));
  if (c->own_stream) cudaStreamDestroy(c->stream);
  if (s) {
    c->stream = reinterpret_cast<cudaStream_t>(s);
    c->own_stream = false;
  } else {
    CK_CTX(c, cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
  }
  return PK_OK;
}

extern "C" int pk_ctx_synchronize(pk_ctx* c) {
  if (!c) return PK_ERR_ARG;
  CK_CTX(c, cudaStreamSynchronize(c->stream));
  return PK_OK;
}

extern "C" int pk_ctx_mem_info(pk_ctx* c, uint64_t* fr, uint64_t* tot, uint64_t* mine) {
  if (!c) return PK_ERR_ARG;
  size_t f = 0, t = 0;
  cudaSetDevice(c->device);
  CK_CTX(c, cudaMemGetInfo(&f, &t));
  if (fr) *fr = f;
  if (tot) *tot = t;
  if (mine) *mine = c->bytes;
  return PK_OK;
}

// ----------------------------------------------------------------- data --
extern "C" int pk_dataset_create(pk_ctx* c, int64_t n, int32_t dim, pk_dataset** out) {
  if (!c || !out || n < 1 || dim < 1) return arg_err(c, "dataset: need n >= 1 and dim >= 1");
  cudaSetDevice(c->device);
  auto* d = new pk_dataset{c, n, dim, nullptr, nullptr};
  const size_t fb = (size_t)n * dim * c->esize();
  cudaError_t e = cudaMalloc(&d->feat, fb);
  if (e == cudaSuccess) e = cudaMalloc((void**)&d->labels, (size_t)n * 4);
  if (e != cudaSuccess) {
    if (d->feat) cudaFree(d->feat);
    delete d;
    c->err = std::string("dataset alloc: ") + cudaGetErrorString(e);
    return PK_ERR_OOM;
  }
  c->bytes += fb + (size_t)n * 4;
  *out = d;
  return PK_OK;
}

extern "C" int pk_dataset_write(pk_dataset* d, int64_t row0, int64_t rows, const double* x,
                                const int64_t* y) {
  if (!d) return PK_ERR_ARG;
  pk_ctx* c = d->ctx;
  if (row0 < 0 || rows < 0 || row0 + rows > d->n || (!x && rows)) return arg_err(c, "dataset_write: bad range");
  if (!rows) return PK_OK;
  cudaSetDevice(c->device);
  const size_t cnt = (size_t)rows * d->dim;
  std::vector<char> hx(cnt * c->esize());
  if (c->dtype == PK_F64) {
    memcpy(hx.data(), x, cnt * 8);
  } else {
    float* f = reinterpret_cast<float*>(hx.data());
    for (size_t i = 0; i < cnt; ++i) f[i] = (float)x[i];
  }
  CK_CTX(c, cudaMemcpyAsync((char*)d->feat + (size_t)row0 * d->dim * c->esize(), hx.data(),
                            hx.size(), cudaMemcpyHostToDevice, c->stream));
  std::vector<int32_t> hy(rows, 0);
  if (y)
    for (int64_t i = 0; i < rows; ++i) hy[i] = (int32_t)y[i];
  CK_CTX(c, cudaMemcpyAsync(d->labels + row0, hy.data(), rows * 4, cudaMemcpyHostToDevice, c->stream));
  CK_CTX(c, cudaStreamSynchronize(c->stream));
  return PK_OK;
}

// device-precision rows straight from (pinned) host memory, enqueued on the
// context stream without a host sync: the streamed-input path of a step
extern "C" int pk_dataset_write_rows(pk_dataset* d, int64_t row0, int64_t rows, const void* x,
                                     const int32_t* y) {
  if (!d) return PK_ERR_ARG;
  pk_ctx* c = d->ctx;
  if (row0 < 0 || rows < 0 || row0 + rows > d->n || (!x && rows) || (!y && rows))
    return arg_err(c, "dataset_write_rows: bad range");
  if (!rows) return PK_OK;
  cudaSetDevice(c->device);
  CK_CTX(c, cudaMemcpyAsync((char*)d->feat + (size_t)row0 * d->dim * c->esize(), x,
                            (size_t)rows * d->dim * c->esize(), cudaMemcpyHostToDevice, c->stream));
  CK_CTX(c, cudaMemcpyAsync(d->labels + row0, y, (size_t)rows * 4, cudaMemcpyHostToDevice,
                            c->stream));
  return PK_OK;
}

// streamed inputs in one call: gather rows idx[0..rows) of a host dataset
// (device precision, row stride src_ld elements) into pinned staging, then
// the same async H2D as pk_dataset_write_rows (the batch gather of
// data.py:131-136, done by memcpy instead of two numpy takes + a copy call)
extern "C" int pk_dataset_gather_rows(pk_dataset* d, int64_t rows, const void* src_x,
                                      int64_t src_ld, const int32_t* src_y, const int64_t* idx,
                                      void* stage_x, int32_t* stage_y) {
  if (!d) return PK_ERR_ARG;
  pk_ctx* c = d->ctx;
  if (rows < 0 || rows > d->n || src_ld < d->dim || (rows && (!src_x || !src_y || !idx ||
                                                              !stage_x || !stage_y)))
    return arg_err(c, "dataset_gather_rows: bad args");
  const size_t es = c->esize(), rb = (size_t)d->dim * es;
  for (int64_t i = 0; i < rows; ++i) {
    memcpy((char*)stage_x + (size_t)i * rb, (const char*)src_x + (size_t)idx[i] * src_ld * es, rb);
    stage_y[i] = src_y[idx[i]];
  }
  return pk_dataset_write_rows(d, 0, rows, stage_x, stage_y);
}

extern "C" int pk_host_map(pk_ctx* c, void* host, int64_t bytes, void** dev) {
  if (!c || !host || bytes <= 0 || !dev) return arg_err(c, "host_map: bad args");
  cudaSetDevice(c->device);
  cudaError_t e = cudaHostRegister(host, (size_t)bytes, cudaHostRegisterMapped);
  if (e == cudaErrorHostMemoryAlreadyRegistered) cudaGetLastError();  // shared buffer: fine
  else CK_CTX(c, e);
  CK_CTX(c, cudaHostGetDevicePointer(dev, host, 0));
  return PK_OK;
}

extern "C" int pk_host_unmap(pk_ctx* c, void* host) {
  if (!c || !host) return PK_ERR_ARG;
  cudaSetDevice(c->device);
  CK_CTX(c, cudaHostUnregister(host));
  return PK_OK;
}

extern "C" int pk_dataset_destroy(pk_dataset* d) {
  if (!d) return PK_ERR_ARG;
  cudaSetDevice(d->ctx->device);
  cudaStreamSynchronize(d->ctx->stream);
  cudaFree(d->feat);
  cudaFree(d->labels);
  d->ctx->bytes -= (size_t)d->n * d->dim * d->ctx->esize() + (size_t)d->n * 4;
  delete d;
  return PK_OK;
}

extern "C" int pk_order_create(pk_ctx* c, const int64_t* perm, int64_t n, pk_order** out) {
  if (!c || !out || !perm || n < 1) return arg_err(c, "order: bad args");
  cudaSetDevice(c->device);
  std::vector<int32_t> h(n);
  for (int64_t i = 0; i < n; ++i) {
    if (perm[i] < 0 || perm[i] >= n) return arg_err(c, "order: index out of range");
    h[i] = (int32_t)perm[i];
  }
  auto* o = new pk_order{c, n, nullptr};
  cudaError_t e = cudaMalloc((void**)&o->perm, (size_t)n * 4);
  if (e != cudaSuccess) {
    delete o;
    c->err = std::string("order alloc: ") + cudaGetErrorString(e);
    return PK_ERR_OOM;
  }
  c->bytes += (size_t)n * 4;
  CK_CTX(c, cudaMemcpyAsync(o->perm, h.data(), (size_t)n * 4, cudaMemcpyHostToDevice, c->stream));
  CK_CTX(c, cudaStreamSynchronize(c->stream));
  *out = o;
  return PK_OK;
}

extern "C" int pk_order_destroy(pk_order* o) {
  if (!o) return PK_ERR_ARG;
  cudaSetDevice(o->ctx->device);
  cudaStreamSynchronize(o->ctx->stream);
  cudaFree(o->perm);
  o->ctx->bytes -= (size_t)o->n * 4;
  delete o;
  return PK_OK;
}

// -------------------------------------------------------------- members --
static int slots_for(int opt) {
  return opt == PK_OPT_SGD ? 0 : (opt == PK_OPT_ADAM ? 2 : 1);
}

extern "C" int pk_member_create(pk_ctx* c, const pk_member_desc* d, pk_member** out) {
  if (!c || !d || !out) return PK_ERR_ARG;
  if (d->n_layers < 1 || d->n_layers > PK_MAX_LAYERS) return arg_err(c, "member: n_layers out of range");
  for (int i = 0; i <= d->n_layers; ++i)
    if (d->dims[i] < 1) return arg_err(c, "member: dims must be >= 1");
  if (d->activation < 0 || d->activation > 3) return arg_err(c, "member: unknown activation");
  if (d->optimizer < 0 || d->optimizer > 3) return arg_err(c, "member: unknown optimizer");
  if (!(d->learning_rate > 0)) return arg_err(c, "member: learning rate must be positive");
  if (d->max_rows < 1) return arg_err(c, "member: max_rows must be >= 1");
  cudaSetDevice(c->device);
  auto* m = new pk_member();
  m->ctx = c;
  m->desc = *d;
  m->n_slots = slots_for(d->optimizer);
  m->m1x = m1x_eligible(*d, c->dtype, c->device);
  m->m1t = !m->m1x && m1t_eligible(*d, c->dtype, c->device);
  m->mlp1 = !m->m1x && !m->m1t && mlp1_eligible(*d, c->dtype, c->device);
  int64_t P = 0;
  for (int l = 0; l < d->n_layers; ++l) {
    m->w_off[l] = P;
    P += (int64_t)d->dims[l] * d->dims[l + 1];
    m->b_off[l] = P;
    P += d->dims[l + 1];
  }
  m->P = P;
  const size_t es = c->esize();
  // slot blocks 32-byte strided: the tensor path's epilogue moves a thread's
  // slots with 256-bit loads/stores (one full sector each)
  m->SS = (int64_t)(align_up((size_t)P * es, 32) / es);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  size_t o_par[2], o_slot[2], o_z[PK_MAX_LAYERS], o_a[PK_MAX_LAYERS], o_dz[PK_MAX_LAYERS];
  for (int b = 0; b < 2; ++b) o_par[b] = take(P * es);
  for (int b = 0; b < 2; ++b) o_slot[b] = take((size_t)m->n_slots * m->SS * es);
  for (int l = 0; l < d->n_layers; ++l) {
    const size_t act = (size_t)d->max_rows * d->dims[l + 1] * es;
    // fused members use Z_1 as the [nb][max_rows][C] partial-logit exchange
    const size_t nb = m->m1t ? (size_t)pk::t_nblk(d->dims[1])
                             : (size_t)(d->dims[1] + pk::M1_BC - 1) / pk::M1_BC;
    o_z[l] = take((m->mlp1 || m->m1t) && l == 1 ? std::max(act, nb * act) : act);
    o_a[l] = take(l + 1 < d->n_layers ? act : 0);
    o_dz[l] = take(act);
  }
  const size_t o_loss = take((size_t)d->max_rows * sizeof(double));
  const size_t o_ctl = take(sizeof(MemberCtl));
  m->slab_bytes = off;
  // recycled from the context when a slab of about this size was freed
  // (Hyperband creates and drops members per configuration; cudaMalloc /
  // cudaFree cost milliseconds at times)
  cudaError_t e = ctx_alloc(c, 0, off, (void**)&m->slab, &m->slab_cap, 1.25);
  if (e != cudaSuccess) {
    delete m;
    c->err = std::string("member alloc: ") + cudaGetErrorString(e);
    return PK_ERR_OOM;
  }
  c->bytes += off;
  for (int b = 0; b < 2; ++b) {
    m->params[b] = m->slab + o_par[b];
    m->slots[b] = m->n_slots ? m->slab + o_slot[b] : nullptr;
  }
  for (int l = 0; l < d->n_layers; ++l) {
    m->Z[l] = m->slab + o_z[l];
    m->A[l] = (l + 1 < d->n_layers) ? m->slab + o_a[l] : nullptr;
    m->dZ[l] = m->slab + o_dz[l];
  }
  m->rowloss = reinterpret_cast<double*>(m->slab + o_loss);
  m->ctl = reinterpret_cast<MemberCtl*>(m->slab + o_ctl);
  CK_CTX(c, cudaMemsetAsync(m->slab, 0, off, c->stream));
  MemberCtl ctl{};
  ctl.parity = 0;
  ctl.bad_node = INT_MAX;
  ctl.bad_grad = INT_MAX;
  ctl.fault_grad = -1;
  ctl.step_counter = 0;
  pk::adam_bias_corrections(0, &ctl.bc1, &ctl.bc2);
  pk::adam_bias_corrections(1, &ctl.bcn1, &ctl.bcn2);
  ctl.lr = d->learning_rate;
  CK_CTX(c, cudaMemcpyAsync(m->ctl, &ctl, sizeof(ctl), cudaMemcpyHostToDevice, c->stream));
  CK_CTX(c, cudaStreamSynchronize(c->stream));
  *out = m;
  return PK_OK;
}

extern "C" int pk_member_destroy(pk_member* m) {
  if (!m) return PK_ERR_ARG;
  cudaSetDevice(m->ctx->device);
  cudaStreamSynchronize(m->ctx->stream);
  ctx_release(m->ctx, 0, m->slab, m->slab_cap);
  m->ctx->bytes -= m->slab_bytes;
  delete m;
  return PK_OK;
}

extern "C" int64_t pk_member_param_count(const pk_member* m) { return m ? m->P : -1; }
extern "C" int32_t pk_member_slot_count(const pk_member* m) { return m ? m->n_slots : -1; }
extern "C" int64_t pk_member_device_bytes(const pk_member* m) { return m ? (int64_t)m->slab_bytes : -1; }

extern "C" int pk_member_set_lr(pk_member* m, double lr) {
  if (!m) return PK_ERR_ARG;
  if (!(lr > 0)) return arg_err(m->ctx, "learning rate must be positive");
  pk_ctx* c = m->ctx;
  cudaSetDevice(c->device);
  m->desc.learning_rate = lr;
  CK_CTX(c, cudaMemcpyAsync(&m->ctl->lr, &m->desc.learning_rate, sizeof(double),
                            cudaMemcpyHostToDevice, c->stream));
  CK_CTX(c, cudaStreamSynchronize(c->stream));
  return PK_OK;
}

extern "C" int pk_member_inject_fault(pk_member* m, int32_t pos) {
  if (!m) return PK_ERR_ARG;
  pk_ctx* c = m->ctx;
  cudaSetDevice(c->device);
  CK_CTX(c, cudaMemcpyAsync(&m->ctl->fault_grad, &pos, sizeof(pos), cudaMemcpyHostToDevice, c->stream));
  CK_CTX(c, cudaStreamSynchronize(c->stream));
  return PK_OK;
}

template <typename T>
static void to_dev_type(const double* src, int64_t n, std::vector<char>& dst) {
  dst.resize(n * sizeof(T));
  T* p = reinterpret_cast<T*>(dst.data());
  for (int64_t i = 0; i < n; ++i) p[i] = (T)src[i];
}

template <typename T>
static void from_dev_type(const std::vector<char>& src, int64_t n, double* dst) {
  const T* p = reinterpret_cast<const T*>(src.data());
  for (int64_t i = 0; i < n; ++i) dst[i] = (double)p[i];
}

extern "C" int pk_member_set_state(pk_member* m, const double* params, const double* slots,
                                   int64_t step_counter) {
  if (!m || !params || step_counter < 0) return PK_ERR_ARG;
  pk_ctx* c = m->ctx;
  cudaSetDevice(c->device);
  CK_CTX(c, cudaStreamSynchronize(c->stream));
  const size_t es = c->esize();
  std::vector<char> hp, hs;
  if (c->dtype == PK_F64) to_dev_type<double>(params, m->P, hp);
  else to_dev_type<float>(params, m->P, hp);
  CK_CTX(c, cudaMemcpyAsync(m->params[0], hp.data(), hp.size(), cudaMemcpyHostToDevice, c->stream));
  if (m->n_slots) {
    const int64_t ns = (int64_t)m->n_slots * m->P;
    CK_CTX(c, cudaMemsetAsync(m->slots[0], 0, (size_t)m->n_slots * m->SS * es, c->stream));
    if (slots) {
      if (c->dtype == PK_F64) to_dev_type<double>(slots, ns, hs);
      else to_dev_type<float>(slots, ns, hs);
      CK_CTX(c, cudaMemcpy2DAsync(m->slots[0], m->SS * es, hs.data(), m->P * es, m->P * es,
                                  m->n_slots, cudaMemcpyHostToDevice, c->stream));
    }
  }
  MemberCtl ctl{};
  CK_CTX(c, cudaMemcpy(&ctl, m->ctl, sizeof(ctl), cudaMemcpyDeviceToHost));  // keeps fault_grad
  ctl.parity = 0;
  ctl.bad_node = INT_MAX;
  ctl.bad_grad = INT_MAX;
  ctl.step_counter = step_counter;
  pk::adam_bias_corrections(step_counter, &ctl.bc1, &ctl.bc2);
  pk::adam_bias_corrections(step_counter + 1, &ctl.bcn1, &ctl.bcn2);
  ctl.lr = m->desc.learning_rate;
  ctl.loss = 0.0;
  ctl.eval_acc = 0.0;
  CK_CTX(c, cudaMemcpyAsync(m->ctl, &ctl, sizeof(ctl), cudaMemcpyHostToDevice, c->stream));
  CK_CTX(c, cudaStreamSynchronize(c->stream));
  return PK_OK;
}

extern "C" int pk_member_get_state(pk_member* m, double* params, double* slots, int64_t* step) {
  if (!m) return PK_ERR_ARG;
  pk_ctx* c = m->ctx;
  cudaSetDevice(c->device);
  CK_CTX(c, cudaStreamSynchronize(c->stream));
  MemberCtl ctl{};
  CK_CTX(c, cudaMemcpy(&ctl, m->ctl, sizeof(ctl), cudaMemcpyDeviceToHost));
  const size_t es = c->esize();
  std::vector<char> h;
  if (params) {
    h.resize(m->P * es);
    CK_CTX(c, cudaMemcpy(h.data(), m->params[ctl.parity], h.size(), cudaMemcpyDeviceToHost));
    if (c->dtype == PK_F64) from_dev_type<double>(h, m->P, params);
    else from_dev_type<float>(h, m->P, params);
  }
  if (slots && m->n_slots) {
    const int64_t ns = (int64_t)m->n_slots * m->P;
    h.resize(ns * es);
    CK_CTX(c, cudaMemcpy2D(h.data(), m->P * es, m->slots[ctl.parity], m->SS * es, m->P * es,
                           m->n_slots, cudaMemcpyDeviceToHost));
    if (c->dtype == PK_F64) from_dev_type<double>(h, ns, slots);
    else from_dev_type<float>(h, ns, slots);
  }
  if (step) *step = ctl.step_counter;
  return PK_OK;
}


// ---------------------------------------------------------------- packs --
#include "pk_pack.cuh"
#include "pk_run.cuh"
