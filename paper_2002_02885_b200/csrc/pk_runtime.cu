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
};

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
  int64_t w_off[PK_MAX_LAYERS], b_off[PK_MAX_LAYERS];
  char* slab;
  size_t slab_bytes;
  void* params[2];
  void* slots[2];
  void* Z[PK_MAX_LAYERS];
  void* A[PK_MAX_LAYERS];
  void* dZ[PK_MAX_LAYERS];
  MemberCtl* ctl;
};

struct Phase {
  int kind;  // 0 fwd, 1 head, 2 bwd, 3 finalize
  Tile* tiles;
  int ntiles;
  int layer;
};

struct Span {
  int kind;
  size_t start;
  int layer;
};

struct pk_pack {
  pk_ctx* ctx;
  std::vector<pk_member*> members;
  int K;
  void* d_members = nullptr;  // MemberDev<T>[K]
  char* d_blob = nullptr;     // StepHdr + FeedDev<T>[K]
  size_t blob_bytes = 0;
  Tile* d_tiles = nullptr;
  std::vector<Phase> phases;
  std::vector<Phase> fwd_phases;  // eval reuses forward + head
  char* h_desc = nullptr;         // pinned ring of descriptors
  char* h_ring = nullptr;         // host-mapped result ring
  char* d_ring = nullptr;
  int32_t ring_stride = 0;
  cudaEvent_t ev[kRing];
  bool ev_pending[kRing];
  int64_t next_ticket = 0;
  cudaGraphExec_t exec = nullptr;
  int launches = 0;
};

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
  int64_t P = 0;
  for (int l = 0; l < d->n_layers; ++l) {
    m->w_off[l] = P;
    P += (int64_t)d->dims[l] * d->dims[l + 1];
    m->b_off[l] = P;
    P += d->dims[l + 1];
  }
  m->P = P;
  const size_t es = c->esize();
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  size_t o_par[2], o_slot[2], o_z[PK_MAX_LAYERS], o_a[PK_MAX_LAYERS], o_dz[PK_MAX_LAYERS];
  for (int b = 0; b < 2; ++b) o_par[b] = take(P * es);
  for (int b = 0; b < 2; ++b) o_slot[b] = take((size_t)m->n_slots * P * es);
  for (int l = 0; l < d->n_layers; ++l) {
    const size_t act = (size_t)d->max_rows * d->dims[l + 1] * es;
    o_z[l] = take(act);
    o_a[l] = take(l + 1 < d->n_layers ? act : 0);
    o_dz[l] = take(act);
  }
  const size_t o_ctl = take(sizeof(MemberCtl));
  m->slab_bytes = off;
  cudaError_t e = cudaMalloc((void**)&m->slab, off);
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
  m->ctl = reinterpret_cast<MemberCtl*>(m->slab + o_ctl);
  CK_CTX(c, cudaMemsetAsync(m->slab, 0, off, c->stream));
  MemberCtl ctl{};
  ctl.parity = 0;
  ctl.bad_node = INT_MAX;
  ctl.bad_grad = INT_MAX;
  ctl.fault_grad = -1;
  ctl.step_counter = 0;
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
  cudaFree(m->slab);
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
    if (slots) {
      if (c->dtype == PK_F64) to_dev_type<double>(slots, ns, hs);
      else to_dev_type<float>(slots, ns, hs);
      CK_CTX(c, cudaMemcpyAsync(m->slots[0], hs.data(), hs.size(), cudaMemcpyHostToDevice, c->stream));
    } else {
      CK_CTX(c, cudaMemsetAsync(m->slots[0], 0, ns * es, c->stream));
    }
  }
  MemberCtl ctl{};
  ctl.parity = 0;
  ctl.bad_node = INT_MAX;
  ctl.bad_grad = INT_MAX;
  ctl.fault_grad = -1;
  ctl.step_counter = step_counter;
  ctl.lr = m->desc.learning_rate;
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
    CK_CTX(c, cudaMemcpy(h.data(), m->slots[ctl.parity], h.size(), cudaMemcpyDeviceToHost));
    if (c->dtype == PK_F64) from_dev_type<double>(h, ns, slots);
    else from_dev_type<float>(h, ns, slots);
  }
  if (step) *step = ctl.step_counter;
  return PK_OK;
}

// ---------------------------------------------------------------- packs --
template <typename T>
static MemberDev<T> member_dev(const pk_member* m) {
  MemberDev<T> d{};
  d.n_layers = m->desc.n_layers;
  d.act = m->desc.activation;
  d.opt = m->desc.optimizer;
  d.max_rows = m->desc.max_rows;
  for (int i = 0; i <= d.n_layers; ++i) d.dims[i] = m->desc.dims[i];
  d.n_slots = m->n_slots;
  d.wd = m->desc.weight_decay;
  d.n_params = m->P;
  for (int l = 0; l < d.n_layers; ++l) {
    d.w_off[l] = m->w_off[l];
    d.b_off[l] = m->b_off[l];
    d.Z[l] = (T*)m->Z[l];
    d.A[l] = (T*)m->A[l];
    d.dZ[l] = (T*)m->dZ[l];
  }
  for (int b = 0; b < 2; ++b) {
    d.params[b] = (T*)m->params[b];
    d.slots[b] = (T*)m->slots[b];
  }
  d.ctl = m->ctl;
  return d;
}

static size_t feed_size(int dtype) {
  return dtype == PK_F64 ? sizeof(FeedDev<double>) : sizeof(FeedDev<float>);
}

// Tile schedule: fixed for the pack's composition and the members' max_rows.
static void build_schedule(pk_pack* p, std::vector<Tile>& all, std::vector<Span>& spans) {
  int lmax = 0;
  for (auto* m : p->members) lmax = std::max(lmax, (int)m->desc.n_layers);
  auto cdiv = [](int a, int b) { return (a + b - 1) / b; };
  // forward phases
  for (int l = 0; l < lmax; ++l) {
    size_t s = all.size();
    for (int k = 0; k < p->K; ++k) {
      const auto& d = p->members[k]->desc;
      if (l >= d.n_layers) continue;
      for (int mb = 0; mb < cdiv(d.max_rows, pk::FWD_BM); ++mb)
        for (int nb = 0; nb < cdiv(d.dims[l + 1], pk::FWD_BN); ++nb)
          all.push_back(Tile{k, (int16_t)l, pk::TK_FWD, mb * pk::FWD_BM, nb * pk::FWD_BN});
    }
    spans.push_back({0, s, l});
  }
  spans.push_back({1, all.size(), lmax - 1});  // head
  for (int l = lmax - 1; l >= 0; --l) {
    size_t s = all.size();
    for (int k = 0; k < p->K; ++k) {
      const auto& d = p->members[k]->desc;
      if (l >= d.n_layers) continue;
      // weight-gradient + update tiles first: they are the long pole
      for (int mb = 0; mb < cdiv(d.dims[l], pk::WG_BM); ++mb)
        for (int nb = 0; nb < cdiv(d.dims[l + 1], pk::WG_BN); ++nb)
          all.push_back(Tile{k, (int16_t)l, pk::TK_WGRAD, mb * pk::WG_BM, nb * pk::WG_BN});
      if (l >= 1)
        for (int mb = 0; mb < cdiv(d.max_rows, pk::DG_BM); ++mb)
          for (int nb = 0; nb < cdiv(d.dims[l], pk::DG_BN); ++nb)
            all.push_back(Tile{k, (int16_t)l, pk::TK_DGRAD, mb * pk::DG_BM, nb * pk::DG_BN});
    }
    spans.push_back({2, s, l});
  }
  spans.push_back({3, all.size(), -1});
}

template <typename T>
static int enqueue_kernels(pk_pack* p, const std::vector<Phase>& phases, int mode) {
  cudaStream_t s = p->ctx->stream;
  const auto* mems = (const MemberDev<T>*)p->d_members;
  const auto* hdr = (const StepHdr*)p->d_blob;
  const auto* feeds = (const FeedDev<T>*)(p->d_blob + sizeof(StepHdr));
  for (const Phase& ph : phases) {
    switch (ph.kind) {
      case 0:
        if (ph.ntiles) pk::k_fwd<T><<<ph.ntiles, pk::NT, 0, s>>>(mems, feeds, ph.tiles);
        break;
      case 1:
        pk::k_head<T><<<p->K, pk::NT, 0, s>>>(mems, feeds, hdr);
        break;
      case 2:
        if (ph.ntiles) pk::k_bwd<T><<<ph.ntiles, pk::NT, 0, s>>>(mems, feeds, ph.tiles);
        break;
      case 3:
        pk::k_finalize<T><<<1, 32, 0, s>>>(mems, feeds, hdr, p->d_ring, p->ring_stride);
        break;
    }
  }
  (void)mode;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    p->ctx->err = std::string("launch: ") + cudaGetErrorString(e);
    return PK_ERR_CUDA;
  }
  return PK_OK;
}

static int enqueue(pk_pack* p, const std::vector<Phase>& ph, int mode) {
  return p->ctx->dtype == PK_F64 ? enqueue_kernels<double>(p, ph, mode)
                                 : enqueue_kernels<float>(p, ph, mode);
}

extern "C" int pk_pack_create(pk_ctx* c, pk_member* const* members, int32_t k, pk_pack** out) {
  if (!c || !out || !members || k < 1) return arg_err(c, "pack needs at least one member");
  cudaSetDevice(c->device);
  for (int i = 0; i < k; ++i) {
    if (!members[i] || members[i]->ctx != c) return arg_err(c, "pack: member from another context");
    for (int j = 0; j < i; ++j)
      if (members[j] == members[i]) return arg_err(c, "pack: duplicate member");
  }
  auto* p = new pk_pack();
  p->ctx = c;
  p->members.assign(members, members + k);
  p->K = k;
  const size_t es = c->esize();
  (void)es;
  // device member table
  size_t mdsz = c->dtype == PK_F64 ? sizeof(MemberDev<double>) : sizeof(MemberDev<float>);
  std::vector<char> hm(mdsz * k);
  for (int i = 0; i < k; ++i) {
    if (c->dtype == PK_F64) {
      auto d = member_dev<double>(members[i]);
      memcpy(hm.data() + i * mdsz, &d, mdsz);
    } else {
      auto d = member_dev<float>(members[i]);
      memcpy(hm.data() + i * mdsz, &d, mdsz);
    }
  }
  std::vector<Tile> tiles;
  std::vector<Span> spans;
  build_schedule(p, tiles, spans);
  p->blob_bytes = sizeof(StepHdr) + feed_size(c->dtype) * k;
  p->ring_stride = (int32_t)align_up(16 + 8 * (size_t)k, 64);
  auto fail = [&](cudaError_t e) {
    c->err = std::string("pack alloc: ") + cudaGetErrorString(e);
    if (p->d_members) cudaFree(p->d_members);
    if (p->d_blob) cudaFree(p->d_blob);
    if (p->d_tiles) cudaFree(p->d_tiles);
    if (p->h_desc) cudaFreeHost(p->h_desc);
    if (p->h_ring) cudaFreeHost(p->h_ring);
    delete p;
    return e == cudaErrorMemoryAllocation ? PK_ERR_OOM : PK_ERR_CUDA;
  };
  cudaError_t e;
  if ((e = cudaMalloc(&p->d_members, hm.size())) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc((void**)&p->d_blob, p->blob_bytes)) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc((void**)&p->d_tiles, std::max<size_t>(1, tiles.size()) * sizeof(Tile))) != cudaSuccess)
    return fail(e);
  if ((e = cudaHostAlloc((void**)&p->h_desc, p->blob_bytes * kRing, cudaHostAllocDefault)) != cudaSuccess)
    return fail(e);
  if ((e = cudaHostAlloc((void**)&p->h_ring, (size_t)p->ring_stride * kRing, cudaHostAllocMapped)) !=
      cudaSuccess)
    return fail(e);
  if ((e = cudaHostGetDevicePointer((void**)&p->d_ring, p->h_ring, 0)) != cudaSuccess) return fail(e);
  memset(p->h_ring, 0, (size_t)p->ring_stride * kRing);
  cudaMemcpyAsync(p->d_members, hm.data(), hm.size(), cudaMemcpyHostToDevice, c->stream);
  if (!tiles.empty())
    cudaMemcpyAsync(p->d_tiles, tiles.data(), tiles.size() * sizeof(Tile), cudaMemcpyHostToDevice, c->stream);
  for (int i = 0; i < kRing; ++i) {
    cudaEventCreateWithFlags(&p->ev[i], cudaEventDisableTiming);
    p->ev_pending[i] = false;
  }
  for (size_t i = 0; i < spans.size(); ++i) {
    const size_t s = spans[i].start;
    const size_t e2 = (i + 1 < spans.size()) ? spans[i + 1].start : tiles.size();
    Phase ph{spans[i].kind, p->d_tiles + s, (int)(e2 - s), spans[i].layer};
    if ((ph.kind == 0 || ph.kind == 2) && ph.ntiles == 0) continue;
    p->phases.push_back(ph);
    if (ph.kind <= 1) p->fwd_phases.push_back(ph);
  }
  p->launches = (int)p->phases.size();
  if ((e = cudaStreamSynchronize(c->stream)) != cudaSuccess) return fail(e);
  c->bytes += hm.size() + p->blob_bytes + tiles.size() * sizeof(Tile);
  *out = p;
  return PK_OK;
}

extern "C" int pk_pack_destroy(pk_pack* p) {
  if (!p) return PK_ERR_ARG;
  pk_ctx* c = p->ctx;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  if (p->exec) cudaGraphExecDestroy(p->exec);
  for (int i = 0; i < kRing; ++i) cudaEventDestroy(p->ev[i]);
  cudaFree(p->d_members);
  cudaFree(p->d_blob);
  cudaFree(p->d_tiles);
  cudaFreeHost(p->h_desc);
  cudaFreeHost(p->h_ring);
  delete p;
  return PK_OK;
}

extern "C" int32_t pk_pack_launches_per_step(const pk_pack* p) { return p ? p->launches : -1; }

template <typename T>
static int fill_feeds(pk_pack* p, const pk_feed* feeds, char* dst) {
  auto* fd = reinterpret_cast<FeedDev<T>*>(dst);
  for (int k = 0; k < p->K; ++k) {
    const pk_feed& f = feeds[k];
    FeedDev<T> d{};
    if (f.take > 0) {
      const pk_member* m = p->members[k];
      if (!f.data) return arg_err(p->ctx, "feed: missing dataset for active member");
      if (f.data->ctx != p->ctx) return arg_err(p->ctx, "feed: dataset from another context");
      if (f.data->dim != m->desc.dims[0]) return arg_err(p->ctx, "feed: dataset dim != member input_dim");
      if (f.take > m->desc.max_rows) return arg_err(p->ctx, "feed: take exceeds member max_rows");
      if (f.pos < 0 || f.pos + f.take > f.data->n) return arg_err(p->ctx, "feed: rows exceed dataset");
      if (f.order && f.order->n != f.data->n) return arg_err(p->ctx, "feed: order length != dataset rows");
      d.feat = (const T*)f.data->feat;
      d.labels = f.data->labels;
      d.rows = f.order ? f.order->perm + f.pos : nullptr;
      d.row0 = f.order ? 0 : f.pos;
      d.ld = f.data->dim;
      d.take = f.take;
    }
    fd[k] = d;
  }
  return PK_OK;
}

static int acquire_slot(pk_pack* p, int64_t ticket, int* slot) {
  const int s = (int)(ticket % kRing);
  if (p->ev_pending[s]) {
    CK_CTX(p->ctx, cudaEventSynchronize(p->ev[s]));
    p->ev_pending[s] = false;
  }
  *slot = s;
  return PK_OK;
}

static int launch_desc(pk_pack* p, int slot, int mode, const pk_feed* feeds) {
  char* h = p->h_desc + (size_t)slot * p->blob_bytes;
  StepHdr hdr{p->K, slot, mode, 0};
  memcpy(h, &hdr, sizeof(hdr));
  int rc = p->ctx->dtype == PK_F64 ? fill_feeds<double>(p, feeds, h + sizeof(StepHdr))
                                   : fill_feeds<float>(p, feeds, h + sizeof(StepHdr));
  if (rc) return rc;
  CK_CTX(p->ctx, cudaMemcpyAsync(p->d_blob, h, p->blob_bytes, cudaMemcpyHostToDevice, p->ctx->stream));
  return PK_OK;
}

extern "C" int pk_pack_step_async(pk_pack* p, const pk_feed* feeds, int64_t* ticket) {
  if (!p || !feeds) return PK_ERR_ARG;
  pk_ctx* c = p->ctx;
  cudaSetDevice(c->device);
  const int64_t t = p->next_ticket;
  int slot;
  int rc = acquire_slot(p, t, &slot);
  if (rc) return rc;
  if ((rc = launch_desc(p, slot, 0, feeds))) return rc;
  if (!p->exec) {
    cudaGraph_t g;
    CK_CTX(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    rc = enqueue(p, p->phases, 0);
    cudaError_t e = cudaStreamEndCapture(c->stream, &g);
    if (rc) return rc;
    CK_CTX(c, e);
    e = cudaGraphInstantiate(&p->exec, g, 0);
    cudaGraphDestroy(g);
    CK_CTX(c, e);
  }
  CK_CTX(c, cudaGraphLaunch(p->exec, c->stream));
  CK_CTX(c, cudaEventRecord(p->ev[slot], c->stream));
  p->ev_pending[slot] = true;
  p->next_ticket = t + 1;
  if (ticket) *ticket = t;
  return PK_OK;
}

static int read_result(pk_pack* p, int slot, double* losses, pk_status* st) {
  const int32_t* s = reinterpret_cast<const int32_t*>(p->h_ring + (size_t)slot * p->ring_stride);
  const double* l = reinterpret_cast<const double*>(s + 4);
  if (st) {
    st->code = s[0];
    st->member = s[1];
    st->index = s[2];
    st->committed = s[3];
  }
  if (losses) memcpy(losses, l, sizeof(double) * p->K);
  return s[0];
}

extern "C" int pk_pack_step_wait(pk_pack* p, int64_t ticket, double* losses, pk_status* st) {
  if (!p || ticket < 0 || ticket >= p->next_ticket || ticket < p->next_ticket - kRing)
    return PK_ERR_STATE;
  pk_ctx* c = p->ctx;
  cudaSetDevice(c->device);
  const int slot = (int)(ticket % kRing);
  if (p->ev_pending[slot]) {
    CK_CTX(c, cudaEventSynchronize(p->ev[slot]));
    p->ev_pending[slot] = false;
  }
  return read_result(p, slot, losses, st);
}

extern "C" int pk_pack_step(pk_pack* p, const pk_feed* feeds, double* losses, pk_status* st) {
  int64_t t;
  int rc = pk_pack_step_async(p, feeds, &t);
  if (rc) return rc;
  return pk_pack_step_wait(p, t, losses, st);
}

extern "C" int pk_pack_eval(pk_pack* p, const pk_dataset* data, const pk_order* order, int64_t pos,
                            int64_t rows, double* losses, pk_status* st) {
  if (!p || !data) return PK_ERR_ARG;
  pk_ctx* c = p->ctx;
  if (rows < 1 || pos < 0 || pos + rows > data->n) return arg_err(c, "eval: bad row range");
  cudaSetDevice(c->device);
  int64_t max_chunks = 0;
  for (auto* m : p->members) max_chunks = std::max<int64_t>(max_chunks, (rows + m->desc.max_rows - 1) / m->desc.max_rows);
  std::vector<pk_feed> feeds(p->K);
  int slot = 0;
  for (int64_t ch = 0; ch < max_chunks; ++ch) {
    for (int k = 0; k < p->K; ++k) {
      const int64_t mr = p->members[k]->desc.max_rows;
      const int64_t off = ch * mr;
      const int64_t tk = std::max<int64_t>(0, std::min<int64_t>(mr, rows - off));
      feeds[k] = pk_feed{data, order, pos + (tk ? off : 0), (int32_t)tk, 0};
    }
    const int64_t t = p->next_ticket++;
    int rc = acquire_slot(p, t, &slot);
    if (rc) return rc;
    if ((rc = launch_desc(p, slot, 1, feeds.data()))) return rc;
    if ((rc = enqueue(p, p->fwd_phases, 1))) return rc;
    CK_CTX(c, cudaEventRecord(p->ev[slot], c->stream));
    p->ev_pending[slot] = true;
  }
  const int64_t t = p->next_ticket++;
  int rc = acquire_slot(p, t, &slot);
  if (rc) return rc;
  if (c->dtype == PK_F64)
    pk::k_eval_finish<double><<<1, 32, 0, c->stream>>>((const MemberDev<double>*)p->d_members, p->K,
                                                         rows, p->d_ring, slot, p->ring_stride);
  else
    pk::k_eval_finish<float><<<1, 32, 0, c->stream>>>((const MemberDev<float>*)p->d_members, p->K,
                                                        rows, p->d_ring, slot, p->ring_stride);
  CK_CTX(c, cudaGetLastError());
  CK_CTX(c, cudaEventRecord(p->ev[slot], c->stream));
  CK_CTX(c, cudaEventSynchronize(p->ev[slot]));
  p->ev_pending[slot] = false;
  return read_result(p, slot, losses, st);
}

extern "C" int pk_pack_profile_step(pk_pack* p, const pk_feed* feeds, float* phase_ms,
                                    int32_t* phase_kind, int32_t* phase_layer,
                                    int32_t* phase_ctas, double* losses, pk_status* st) {
  if (!p || !feeds) return PK_ERR_ARG;
  pk_ctx* c = p->ctx;
  cudaSetDevice(c->device);
  const int64_t t = p->next_ticket++;
  int slot;
  int rc = acquire_slot(p, t, &slot);
  if (rc) return rc;
  if ((rc = launch_desc(p, slot, 0, feeds))) return rc;
  const int n = (int)p->phases.size();
  std::vector<cudaEvent_t> ev(n + 1);
  for (auto& e : ev) CK_CTX(c, cudaEventCreate(&e));
  for (int i = 0; i < n; ++i) {
    CK_CTX(c, cudaEventRecord(ev[i], c->stream));
    std::vector<Phase> one{p->phases[i]};
    if ((rc = enqueue(p, one, 0))) return rc;
  }
  CK_CTX(c, cudaEventRecord(ev[n], c->stream));
  CK_CTX(c, cudaEventSynchronize(ev[n]));
  for (int i = 0; i < n; ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
    const Phase& ph = p->phases[i];
    if (phase_ms) phase_ms[i] = ms;
    if (phase_kind) phase_kind[i] = ph.kind;
    if (phase_layer) phase_layer[i] = ph.layer;
    if (phase_ctas) phase_ctas[i] = ph.kind == 1 ? p->K : (ph.kind == 3 ? 1 : ph.ntiles);
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return read_result(p, slot, losses, st);
}
