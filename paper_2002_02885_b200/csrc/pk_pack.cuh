// pk_pack.cuh — the pack half of the runtime (included by pk_runtime.cu so
// the whole library is one translation unit).
//
// A pack is an ordered list of members.  Its packed step is a fixed
// schedule of phases built once from the members' shapes:
//
//   member stages:  FWD(0) .. FWD(L-1) | TAIL                 (or FWD(L), HEAD, DGRAD(L))
//                   | WGRAD(L) WGRAD(L-1) DGRAD(L-1) | WGRAD(L-2) DGRAD(L-2) | .. | WGRAD(0)
//   phase p      =  stage p of every member (one grouped launch of k_phase)
//
// Phases are launched with programmatic dependent launch and captured once
// into a CUDA graph; a step is then one H2D descriptor copy + one graph
// launch.  The last CTA of the last phase runs FINALIZE and writes
// {status, losses} into a host-mapped ring slot.

#pragma once

struct Phase {
  std::vector<Tile> host;  // tiles (host copy, for schedule inspection)
  Tile* tiles = nullptr;   // device copy
  int ntiles = 0;
  int smem = 0;            // dynamic shared memory bytes
  int kind = 0;            // dominant tile kind (reporting)
  int mask = 0;            // OR of (1 << tile kind) present → which kernel
  int special = 0;         // 0 phase kernel, 1 k_mlp1_fwd, 2 k_mlp1_bwd, 3 k_m1t_fwd, 4 k_m1t_bwd,
                           // 5 k_m1s_fwd, 6 k_m1c_fwd, 7 k_m1x_step
  int layer = -1;          // dominant layer (reporting)
  int cs = 1;              // thread-block cluster size (k_m1t_fwd)
  int stages = 1;          // k_m1t_bwd input-tile stages
  int gsize = 1;           // k_m1t_bwd input tiles per group
  int nt = pk::NT;         // threads per CTA
};

struct pk_pack {
  pk_ctx* ctx;
  std::vector<pk_member*> members;
  int K;
  void* d_members = nullptr;  // MemberDev<T>[K]
  char* d_blob = nullptr;     // StepHdr + FeedDev<T>[K]
  size_t blob_bytes = 0;
  int32_t* d_done = nullptr;  // CTA-completion counter for FINALIZE (+ FWD split workspace)
  size_t done_bytes = 16;
  unsigned long long* d_trace = nullptr;  // PK_TRACE=1: stage stamps per CTA
  size_t trace_len = 0;
  Tile* d_tiles = nullptr;
  std::vector<Phase> train;   // phases of a train step
  std::vector<Phase> eval;    // forward-only phases (validation loss)
  char* h_desc = nullptr;     // pinned ring of descriptors
  char* h_ring = nullptr;     // host-mapped result ring
  char* d_ring = nullptr;
  int32_t ring_stride = 0;
  cudaEvent_t ev[kRing];
  bool ev_pending[kRing];
  int64_t next_ticket = 0;
  cudaGraphExec_t exec = nullptr;
  // inline step descriptors (K <= kInlineFeeds): the train graph's kernel
  // nodes, re-parameterised every step instead of copying a descriptor H2D
  struct Node {
    cudaGraphNode_t node;
    cudaKernelNodeParams kp;
    std::vector<char> args;  // PhaseArgs<T> bytes
  };
  bool inline_desc = false;
  cudaGraph_t graph = nullptr;
  std::vector<Node> nodes;
  std::vector<char> h_feeds;  // host FeedDev<T>[K] of the step being launched
  std::vector<char> h_mems;   // host MemberDev<T>[K] (static)
  bool halt_dirty = false;    // a failed step set the device halt flag
  struct RunStage {           // pk_pack_run's streamed-input slot (pinned + device)
    pk_dataset* d = nullptr;
    void* hx = nullptr;
    int32_t* hy = nullptr;
  };
  std::vector<RunStage> run_stage;
  // pk_pack_run's streamed inputs travel on their own stream, so step n+1's
  // H2D overlaps step n's kernels; the pack stream waits on ev_copy[slot]
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copy[kRing] = {};
  // pk_pack_run's multi-step graph: `multi_n` whole steps captured back to
  // back, each step's first launch chained to the previous step by PDL
  int multi_n = 0;
  cudaGraph_t graph_multi = nullptr;
  cudaGraphExec_t exec_multi = nullptr;
  std::vector<std::vector<Node>> nodes_multi;
  // capacities of the recycled context blocks this pack holds
  size_t cap_members = 0, cap_blob = 0, cap_done = 0, cap_tiles = 0, cap_desc = 0, cap_ring = 0;
};

template <typename T>
static MemberDev<T> member_dev(const pk_member* m, int tail) {
  MemberDev<T> d{};
  d.n_layers = m->desc.n_layers;
  d.act = m->desc.activation;
  d.opt = m->desc.optimizer;
  d.max_rows = m->desc.max_rows;
  for (int i = 0; i <= d.n_layers; ++i) d.dims[i] = m->desc.dims[i];
  d.n_slots = m->n_slots;
  d.tail = tail;
  d.tensor = (m->m1t || m->m1x) ? 1 : 0;
  d.wd = m->desc.weight_decay;
  d.n_params = m->P;
  d.s_stride = m->SS;
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
  d.rowloss = m->rowloss;
  d.ctl = m->ctl;

  return d;
}

static size_t feed_size(int dtype) {
  return dtype == PK_F64 ? sizeof(FeedDev<double>) : sizeof(FeedDev<float>);
}

// dynamic shared memory a k_phase CTA may use (opt-in limit minus the
// kernel's static smem), set once per precision by pk_pack_create
// the process-wide kernel plan (packtrain_b200.h pk_plan_options)
static pk_plan_options plan_defaults() {
  pk_plan_options o;
  memset(&o, 0, sizeof(o));
  o.tcgen05 = o.mlp1 = o.fwd_split = o.wgrad_narrow = o.inline_desc = o.conv_cluster = 1;
  o.conv_halo = 1;
  return o;
}
static pk_plan_options g_plan = plan_defaults();

static int g_smem_max[2] = {0, 0};

static int smem_budget(int dtype) { return g_smem_max[dtype]; }

template <typename T>
using PhaseKernel = void (*)(const pk::PhaseArgs<T>);

// the lean kernel for a phase's kind mask (see KM_* in pk_kernels.cuh)
template <typename T>
static PhaseKernel<T> kernel_for(int mask) {
  switch (mask) {
    case pk::KM_FWD: return pk::k_phase<T, pk::KM_FWD>;
    case pk::KM_TAIL: return pk::k_phase<T, pk::KM_TAIL>;
    case pk::KM_HEAD: return pk::k_phase<T, pk::KM_HEAD>;
    case pk::KM_DGRAD: return pk::k_phase<T, pk::KM_DGRAD>;
    case pk::KM_WGRAD: return pk::k_phase<T, pk::KM_WGRAD>;
    case pk::KM_WGRAD | pk::KM_DGRAD: return pk::k_phase<T, pk::KM_WGRAD | pk::KM_DGRAD>;
    default: return pk::k_phase<T, pk::KM_ALL>;
  }
}

template <typename T>
static cudaError_t init_smem_limit(int device, int* out) {
  int optin = 0;
  cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (e != cudaSuccess) return e;
  const int masks[] = {pk::KM_FWD, pk::KM_TAIL, pk::KM_HEAD, pk::KM_DGRAD, pk::KM_WGRAD,
                       pk::KM_WGRAD | pk::KM_DGRAD, pk::KM_ALL};
  std::vector<PhaseKernel<T>> ks;
  for (int mk : masks) ks.push_back(kernel_for<T>(mk));
  ks.push_back(pk::k_mlp1_fwd<T>);
  ks.push_back(pk::k_mlp1_bwd<T>);
  ks.push_back(pk::k_m1t_fwd<T>);
  ks.push_back(pk::k_m1t_bwd<T>);
  ks.push_back(pk::k_m1s_fwd<T>);
  ks.push_back(pk::k_m1c_fwd<T>);
  ks.push_back(pk::k_m1x_step<T>);
  int dyn = optin;
  for (auto k : ks) {
    cudaFuncAttributes fa{};
    if ((e = cudaFuncGetAttributes(&fa, k)) != cudaSuccess) return e;
    dyn = std::min(dyn, optin - (int)fa.sharedSizeBytes);
  }
  for (auto k : ks)
    if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn)) !=
        cudaSuccess)
      return e;
  // input-split clusters of k_m1t_fwd go up to 16 CTAs (non-portable size)
  if ((e = cudaFuncSetAttribute(pk::k_m1t_fwd<T>, cudaFuncAttributeNonPortableClusterSizeAllowed,
                                1)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(pk::k_m1c_fwd<T>, cudaFuncAttributeNonPortableClusterSizeAllowed,
                                1)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(pk::k_m1x_step<T>, cudaFuncAttributeNonPortableClusterSizeAllowed,
                                1)) != cudaSuccess)
    return e;
  *out = dyn;
  return e;
}

static int cdiv(int a, int b) { return (a + b - 1) / b; }

// conservative dynamic-smem budget for member-level decisions (made before
// any pack exists): the opt-in limit minus a margin for static smem
constexpr int kStaticSmemMargin = 16 * 1024;

static bool mlp1_eligible(const pk_member_desc& d, int dtype, int device) {
  if (d.n_layers != 2 || d.dims[2] > pk::M1_MAXC || d.max_rows > pk::M1_MAXR) return false;
  if (!g_plan.mlp1) return false;
  // f64 members: the phase kernels are faster at every Hyperband shape
  // (784-16-10: 45 vs 78 µs per step at K=1, 74 vs 128 at K=8 — its 8-unit
  // column blocks leave a narrow member with 2 CTAs walking all 784 inputs)
  if (dtype == PK_F64) return false;
  int optin = 0;
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) !=
      cudaSuccess)
    return false;
  const int budget = optin - kStaticSmemMargin;
  const int D = d.dims[0], C = d.dims[2], RP = pk::m1_rows_pad(d.max_rows);
  const int ns = d.optimizer == PK_OPT_SGD ? 0 : (d.optimizer == PK_OPT_ADAM ? 2 : 1);
  const bool f64 = dtype == PK_F64;
  const int fs = f64 ? pk::M1<double>::fwd_smem(D, C, RP) : pk::M1<float>::fwd_smem(D, C, RP);
  const int bs = f64 ? pk::M1<double>::bwd_smem(D, C, RP, ns) : pk::M1<float>::bwd_smem(D, C, RP, ns);
  return fs <= budget && bs <= budget;
}

// tensor-core path (pk_m1t.cuh): fp32, one hidden layer, <= 32 classes,
// <= 128 rows, 16-byte aligned W0 rows / dataset rows for the bulk copies
static bool m1t_eligible(const pk_member_desc& d, int dtype, int device) {
  if (dtype != PK_F32 || d.n_layers != 2) return false;
  const int D = d.dims[0], H = d.dims[1], C = d.dims[2];
  if (C > pk::T_MAXC || d.max_rows > pk::T_MAXR || H % 4 != 0 || D % 4 != 0) return false;
  if (pk::t_nsplit(D) > pk::T_MAXCS) return false;  // one cluster per unit tile
  if (!g_plan.tcgen05) return false;
  int optin = 0;
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) !=
      cudaSuccess)
    return false;
  const int budget = optin - kStaticSmemMargin;
  const int RP = pk::m1_rows_pad(d.max_rows);
  const int ns = d.optimizer == PK_OPT_SGD ? 0 : (d.optimizer == PK_OPT_ADAM ? 2 : 1);
  return pk::M1T::fwd_smem(RP, C) <= budget && pk::M1T::bwd_smem(RP, C, ns, 1) <= budget;
}

// one-launch cluster step (pk_m1x.cuh): the largest 16-unit blocks per CTA
// (1, 2, 4) the register tiling and `budget` bytes of smem allow, 0 if none
static int x_bpc_hi(const pk_member_desc& d, int ns, int budget) {
  const int RP = pk::m1_rows_pad(d.max_rows), C = d.dims[2];
  for (int b = pk::x_bpc_max(RP); b >= 1; b /= 2)
    if (pk::M1X::smem(RP, pk::X_UB * b, C, ns, 2) <= budget) return b;
  return 0;
}

// fp32, one hidden layer, <= 32 classes, <= 64 rows, 16-byte aligned rows,
// and one cluster (<= 16 CTAs) covers the hidden layer
static bool m1x_eligible(const pk_member_desc& d, int dtype, int device) {
  if (dtype != PK_F32 || d.n_layers != 2) return false;
  const int D = d.dims[0], H = d.dims[1], C = d.dims[2];
  if (C > pk::X_MAXC || d.max_rows > pk::X_MAXR || H % 4 != 0 || D % 4 != 0) return false;
  // opt-in while its step time trails the tcgen05 path's (plan option m1x)
  if (!g_plan.m1x) return false;
  int optin = 0;
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) !=
      cudaSuccess)
    return false;
  const int ns = d.optimizer == PK_OPT_SGD ? 0 : (d.optimizer == PK_OPT_ADAM ? 2 : 1);
  const int b = x_bpc_hi(d, ns, optin - kStaticSmemMargin);
  return b > 0 && cdiv(pk::x_nblk(H), b) <= pk::X_MAXCS;
}

// whether the member's last layer + head + first dgrad fit one TAIL tile
static bool tail_ok(const pk_member* m, int dtype) {
  const int L = m->desc.n_layers - 1;
  const int in = m->desc.dims[L], C = m->desc.dims[L + 1];
  if (C > pk::TAIL_MAXC) return false;
  const int need = dtype == PK_F64 ? pk::Smem<double>::tail(in, C) : pk::Smem<float>::tail(in, C);
  return need <= smem_budget(dtype);
}

static int kind_smem(int kind, const pk_member* m, int dtype) {
  const bool d = dtype == PK_F64;
  const int L = m->desc.n_layers - 1;
  switch (kind) {
    case pk::TK_FWD: return d ? pk::Smem<double>::FWD : pk::Smem<float>::FWD;
    case pk::TK_TAIL:
      return d ? pk::Smem<double>::tail(m->desc.dims[L], m->desc.dims[L + 1])
               : pk::Smem<float>::tail(m->desc.dims[L], m->desc.dims[L + 1]);
    case pk::TK_HEAD: return d ? pk::Smem<double>::HEAD : pk::Smem<float>::HEAD;
    case pk::TK_DGRAD: return d ? pk::Smem<double>::DGRAD : pk::Smem<float>::DGRAD;
    default: return d ? pk::Smem<double>::WGRAD : pk::Smem<float>::WGRAD;
  }
}


// tiles of one (member, kind, layer) work item
static void emit(std::vector<Tile>& out, int k, const pk_member* m, int kind, int l,
                 int fwd_ctas = 1) {
  const auto& d = m->desc;
  switch (kind) {
    case pk::TK_FWD: {
      // input ranges from the member's shape alone (pk_kernels.cuh fwd_tile);
      // CTAs per tile (ng) from the phase's room, which never changes the sums
      const int nch = cdiv(d.dims[l], pk::FWD_KC);
      int cps = 0, nr = 1;
      if (nch >= 3 && g_plan.fwd_split) {
        cps = std::max(2, cdiv(nch, pk::kFwdMaxRanges));
        nr = cdiv(nch, cps);
        if (cps > 127) cps = 0, nr = 1;
      }
      const int ng = std::max(1, std::min({nr, fwd_ctas, 16}));
      for (int mb = 0; mb < cdiv(d.max_rows, pk::FWD_BM); ++mb)
        for (int nb = 0; nb < cdiv(d.dims[l + 1], pk::FWD_BN); ++nb)
          for (int g = 0; g < ng; ++g)
            out.push_back(Tile{k, (int16_t)l, (int16_t)kind,
                               pk::fwd_pack_m0(mb * pk::FWD_BM, g, ng),
                               pk::fwd_pack_n0(nb * pk::FWD_BN, cps)});
      break;
    }
    case pk::TK_TAIL:
      for (int mb = 0; mb < cdiv(d.max_rows, pk::TAIL_BM); ++mb)
        out.push_back(Tile{k, (int16_t)l, (int16_t)kind, mb * pk::TAIL_BM, 0});
      break;
    case pk::TK_HEAD:
      for (int mb = 0; mb < cdiv(d.max_rows, pk::HEAD_BM); ++mb)
        out.push_back(Tile{k, (int16_t)l, (int16_t)kind, mb * pk::HEAD_BM, 0});
      break;
    case pk::TK_DGRAD:
      for (int mb = 0; mb < cdiv(d.max_rows, pk::DG_BM); ++mb)
        for (int nb = 0; nb < cdiv(d.dims[l], pk::DG_BN); ++nb)
          out.push_back(Tile{k, (int16_t)l, (int16_t)kind, mb * pk::DG_BM, nb * pk::DG_BN});
      break;
    default:  // WGRAD over W_l [in x out]
      if (d.dims[l + 1] <= pk::WGN_BN && g_plan.wgrad_narrow) {
        // narrow layer: 64 x 16 tiles (pk_kernels.cuh WgradNG), flagged by n0 bit 20
        for (int mb = 0; mb < cdiv(d.dims[l], pk::WGN_BM); ++mb)
          out.push_back(Tile{k, (int16_t)l, (int16_t)kind, mb * pk::WGN_BM, 1 << 20});
        break;
      }
      for (int mb = 0; mb < cdiv(d.dims[l], pk::WG_BM); ++mb)
        for (int nb = 0; nb < cdiv(d.dims[l + 1], pk::WG_BN); ++nb)
          out.push_back(Tile{k, (int16_t)l, (int16_t)kind, mb * pk::WG_BM, nb * pk::WG_BN});
      break;
  }
}

using Stage = std::vector<std::pair<int, int>>;  // (kind, layer)

// per-member stage sequence; `fwd_stages` = how many form the forward pass
static std::vector<Stage> member_stages(const pk_member* m, bool tail, int* fwd_stages) {
  const int L = m->desc.n_layers - 1;
  std::vector<Stage> st;
  for (int l = 0; l < L; ++l) st.push_back({{pk::TK_FWD, l}});
  if (tail) {
    st.push_back({{pk::TK_TAIL, L}});
    *fwd_stages = (int)st.size();
  } else {
    st.push_back({{pk::TK_FWD, L}});
    st.push_back({{pk::TK_HEAD, L}});
    *fwd_stages = (int)st.size();
    if (L >= 1) st.push_back({{pk::TK_DGRAD, L}});
  }
  if (L == 0) {
    st.push_back({{pk::TK_WGRAD, 0}});
  } else {
    Stage s{{pk::TK_WGRAD, L}, {pk::TK_WGRAD, L - 1}};
    if (L - 1 >= 1) s.push_back({pk::TK_DGRAD, L - 1});
    st.push_back(s);
    for (int l = L - 2; l >= 0; --l) {
      Stage s2{{pk::TK_WGRAD, l}};
      if (l >= 1) s2.push_back({pk::TK_DGRAD, l});
      st.push_back(s2);
    }
  }
  return st;
}

// k_m1x_step: one cluster of CS CTAs per member; member k's CTAs own
// bpc_k = pow2 >= nblk_k / CS unit blocks each.  CS is the largest cluster
// size whose clusters all run co-resident (one wave); the arithmetic does not
// depend on it (pk_m1x.cuh), so packed == standalone still holds bitwise.
static Phase build_m1x_phase(pk_pack* p) {
  Phase xs;
  xs.special = 7;
  xs.kind = pk::TK_FWD;
  xs.layer = 0;
  std::vector<int> xm;
  for (int k = 0; k < p->K; ++k)
    if (p->members[k]->m1x) xm.push_back(k);
  if (xm.empty()) return xs;
  const int dt = p->ctx->dtype, budget = smem_budget(dt);
  auto nblk = [&](int k) { return pk::x_nblk(p->members[k]->desc.dims[1]); };
  auto plan = [&](int CS, std::vector<int>& bpc, int* Sb, int* sm) {
    bpc.assign(p->K, 0);
    for (int k : xm) {
      const pk_member* m = p->members[k];
      int b = 1;
      while (b * CS < nblk(k)) b *= 2;
      if (b > x_bpc_hi(m->desc, m->n_slots, budget)) return false;
      bpc[k] = b;
    }
    for (*Sb = 4; *Sb >= 2; --*Sb) {
      *sm = 0;
      for (int k : xm) {
        const pk_member* m = p->members[k];
        *sm = std::max(*sm, pk::M1X::smem(pk::m1_rows_pad(m->desc.max_rows), pk::X_UB * bpc[k],
                                          m->desc.dims[2], m->n_slots, *Sb));
      }
      if (*sm <= budget) return true;
    }
    return false;
  };
  // candidate cluster sizes: every member's nblk / {1, 2, 4}, largest first
  std::vector<int> cand;
  for (int k : xm)
    for (int b = 1; b <= 4; b *= 2) {
      const int cs = cdiv(nblk(k), b);
      if (cs <= pk::X_MAXCS) cand.push_back(cs);
    }
  std::sort(cand.rbegin(), cand.rend());
  cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
  int CS = 0, Sb = 2, sm = 0;
  std::vector<int> bpc;
  for (int cs : cand) {
    int sb, s;
    std::vector<int> b;
    if (!plan(cs, b, &sb, &s)) continue;
    if (!CS || cs < CS) { CS = cs; Sb = sb; sm = s; bpc = b; }  // fallback: fewest CTAs
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cs * (int)xm.size());
    cfg.blockDim = dim3(pk::NT);
    cfg.dynamicSmemBytes = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, pk::k_m1x_step<float>, &cfg) == cudaSuccess &&
        nc >= (int)xm.size()) {
      CS = cs; Sb = sb; sm = s; bpc = b;
      break;
    }
  }
  cudaGetLastError();  // an occupancy query error is not sticky for the caller
  if (!CS) return xs;  // cannot happen for eligible members; fall through empty
  for (int k : xm)
    for (int r = 0; r < CS; ++r) xs.host.push_back(Tile{k, (int16_t)bpc[k], pk::TK_FWD, r, 0});
  xs.cs = CS;
  xs.stages = Sb;

  xs.smem = sm;
  xs.ntiles = (int)xs.host.size();
  return xs;
}

static void build_phases(pk_pack* p, bool eval, std::vector<Phase>& phases) {
  const int dt = p->ctx->dtype;
  std::vector<std::vector<Stage>> seq(p->K);
  size_t nph = 0;
  Phase m1f, m1b;  // fused one-hidden-layer members (train only)
  m1f.special = 1;
  m1b.special = 2;
  Phase tf, tb;    // tensor-core one-hidden-layer members (train only)
  tf.special = 3;
  tb.special = 4;
  tb.nt = pk::T_BWD_NT;
  // k_m1t_fwd: one cluster (= all input splits) per unit tile.  k_m1t_bwd: a
  // CTA per (unit tile, group of G input tiles), G sized for ~one wave; two
  // input-tile stages in flight when every member's shared memory allows.
  int n_ut = 0, n_kt = 1;
  tb.stages = 4;  // input-tile stages (the kernel may use more if its member allows)
  for (int k = 0; k < p->K; ++k) {
    const pk_member* m = p->members[k];
    if (eval || !m->m1t) continue;
    tf.cs = std::max(tf.cs, pk::t_nsplit(m->desc.dims[0]));
    n_ut += cdiv(m->desc.dims[1], pk::T_BU);
    n_kt = std::max(n_kt, cdiv(m->desc.dims[0], pk::T_BK));
    while (tb.stages > 1 &&
           pk::M1T::bwd_smem(pk::m1_rows_pad(m->desc.max_rows), m->desc.dims[2], m->n_slots,
                             tb.stages) > smem_budget(dt))
      --tb.stages;
  }
  const int G = std::max(1, std::min(n_kt, cdiv(n_ut * n_kt, 148)));
  tb.gsize = G;
  for (int k = 0; k < p->K; ++k) {
    const pk_member* m = p->members[k];
    if (!eval && m->m1x) continue;  // the one-launch cluster step, below
    if (!eval && m->m1t) {
      const int D = m->desc.dims[0], H = m->desc.dims[1], C = m->desc.dims[2];
      const int RP = pk::m1_rows_pad(m->desc.max_rows);
      for (int t = 0; t < pk::t_ntile(H); ++t)
        for (int s = 0; s < tf.cs; ++s) tf.host.push_back(Tile{k, 0, pk::TK_FWD, t, s});
      const int nkt = cdiv(D, pk::T_BK);
      for (int ut = 0; ut < cdiv(H, pk::T_BU); ++ut)
        for (int kt = 0; kt < nkt; kt += G)
          tb.host.push_back(Tile{k, (int16_t)std::min(G, nkt - kt), pk::TK_WGRAD, kt, ut});
      tf.smem = std::max(tf.smem, pk::M1T::fwd_smem(RP, C));
      tb.smem = std::max(tb.smem, pk::M1T::bwd_smem(RP, C, m->n_slots, tb.stages));
      continue;
    }
    if (!eval && m->mlp1) {
      const int nb = (m->desc.dims[1] + pk::M1_BC - 1) / pk::M1_BC;
      for (int cb = 0; cb < nb; ++cb) m1f.host.push_back(Tile{k, 0, pk::TK_FWD, cb, 0});
      const int D = m->desc.dims[0], C = m->desc.dims[2], RP = pk::m1_rows_pad(m->desc.max_rows);
      const bool f64 = dt == PK_F64;
      m1f.smem = std::max(m1f.smem, f64 ? pk::M1<double>::fwd_smem(D, C, RP)
                                        : pk::M1<float>::fwd_smem(D, C, RP));
      m1b.smem = std::max(m1b.smem, f64 ? pk::M1<double>::bwd_smem(D, C, RP, m->n_slots)
                                        : pk::M1<float>::bwd_smem(D, C, RP, m->n_slots));
      continue;
    }
    int nf = 0;
    seq[k] = member_stages(m, tail_ok(m, dt), &nf);
    if (eval) seq[k].resize(nf);
    nph = std::max(nph, seq[k].size());
  }
  m1f.ntiles = (int)m1f.host.size();
  m1b.host = m1f.host;
  m1b.ntiles = m1f.ntiles;
  m1f.kind = m1b.kind = pk::TK_FWD;
  m1f.layer = 0;
  m1b.layer = 1;
  phases.assign(nph, Phase{});
  for (size_t ph = 0; ph < nph; ++ph) {
    Phase& P = phases[ph];
    double best = -1;
    // FWD tiles share a tile among up to (SMs / tiles of the phase) CTAs
    std::vector<Tile> probe;
    for (int k = 0; k < p->K; ++k)
      if (ph < seq[k].size())
        for (auto [kind, layer] : seq[k][ph]) emit(probe, k, p->members[k], kind, layer);
    const int fwd_ctas = std::max(1, 148 / std::max<int>(1, (int)probe.size()));
    for (int k = 0; k < p->K; ++k) {
      if (ph >= seq[k].size()) continue;
      for (auto [kind, layer] : seq[k][ph]) {
        const size_t before = P.host.size();
        emit(P.host, k, p->members[k], kind, layer, fwd_ctas);
        P.smem = std::max(P.smem, kind_smem(kind, p->members[k], dt));
        const double w = double(P.host.size() - before);
        if (w > best) { best = w; P.kind = kind; P.layer = layer; }
        P.mask |= 1 << kind;
      }
    }
    P.ntiles = (int)P.host.size();
  }
  if (m1f.ntiles) {
    phases.insert(phases.begin(), m1f);
    phases.push_back(m1b);
  }
  // default forward: cluster-streaming (k_m1c_fwd) with the cluster size that
  // fills about one wave; plan option fwd = 1 | 2 pins the other variants
  if (!eval && !tf.host.empty() && g_plan.fwd == 0) {
    int n_tiles = 0, cs_lo = 1, ns_max = 1, sm = 0;
    for (int k = 0; k < p->K; ++k) {
      const pk_member* m = p->members[k];
      if (!m->m1t) continue;
      const int RP = pk::m1_rows_pad(m->desc.max_rows), ns = pk::t_nsplit(m->desc.dims[0]);
      n_tiles += pk::t_ntile(m->desc.dims[1]);
      cs_lo = std::max(cs_lo, cdiv(ns, pk::m1c_max_local(RP)));
      ns_max = std::max(ns_max, ns);
      sm = std::max(sm, pk::m1c_fwd_smem(RP, m->desc.dims[2]));
    }
    // the largest cluster size whose clusters all fit co-resident (one
    // wave); never below what TMEM / smem per CTA allow
    int CS = cs_lo;
    bool one_wave = false;
    int cs_hi = std::min(ns_max, pk::T_MAXCS);
    if (g_plan.fwd_cluster > 0) cs_hi = std::max(cs_lo, std::min(cs_hi, g_plan.fwd_cluster));
    for (int cs = cs_hi; cs >= cs_lo; --cs) {
      if (dt != PK_F32) break;
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(cs * n_tiles);
      cfg.blockDim = dim3(pk::NT);
      cfg.dynamicSmemBytes = sm;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int nc = 0;
      if (cudaOccupancyMaxActiveClusters(&nc, pk::k_m1c_fwd<float>, &cfg) == cudaSuccess &&
          nc >= n_tiles) {
        CS = cs;
        one_wave = true;
        break;
      }
    }
    // one split per CTA fits in a wave: the one-shot split-K cluster forward
    // (same arithmetic, no streaming pipeline) is the lower-latency choice.
    // No cluster size fits a wave (many unit tiles): one streaming CTA per
    // tile (k_m1s_fwd, below) instead.
    if (one_wave && CS < ns_max && sm <= smem_budget(dt)) {
      tf.host.clear();
      for (int k = 0; k < p->K; ++k)
        if (p->members[k]->m1t)
          for (int t = 0; t < pk::t_ntile(p->members[k]->desc.dims[1]); ++t)
            for (int r = 0; r < CS; ++r) tf.host.push_back(Tile{k, 0, pk::TK_FWD, t, r});
      tf.special = 6;
      tf.cs = CS;
      tf.smem = sm;
    }
  }
  // many clusters (several waves): stream the input dimension instead, one CTA
  // per unit tile, when every tensor member's streaming smem fits
  if (!eval && tf.special == 3 && g_plan.fwd != 1 &&
      ((int)tf.host.size() > 2 * 148 || g_plan.fwd == 2)) {
    // (also reached when no m1c cluster size fits a wave)
    bool fits = true;
    int sm = 0;
    for (int k = 0; k < p->K; ++k) {
      const pk_member* m = p->members[k];
      if (!m->m1t) continue;
      const int need = pk::m1s_fwd_smem(pk::m1_rows_pad(m->desc.max_rows), m->desc.dims[2]);
      fits &= need <= smem_budget(dt);
      sm = std::max(sm, need);
    }
    if (fits) {
      tf.host.clear();
      for (int k = 0; k < p->K; ++k)
        if (p->members[k]->m1t)
          for (int t = 0; t < pk::t_ntile(p->members[k]->desc.dims[1]); ++t)
            tf.host.push_back(Tile{k, 0, pk::TK_FWD, t, 0});
      tf.special = 5;
      tf.cs = 1;
      tf.smem = sm;
    }
  }
  tf.ntiles = (int)tf.host.size();
  tb.ntiles = (int)tb.host.size();
  tf.kind = pk::TK_FWD;
  tb.kind = pk::TK_WGRAD;
  tf.layer = 0;
  tb.layer = 0;
  if (tf.ntiles) {
    phases.insert(phases.begin(), tf);
    phases.push_back(tb);
  }
  if (!eval) {
    Phase xs = build_m1x_phase(p);
    if (xs.ntiles) phases.insert(phases.begin(), xs);
  }
}

// only >= 0: launch that phase alone (profiling); finalize: let the last
// launch run FINALIZE
template <typename T>
static int launch_phases(pk_pack* p, const std::vector<Phase>& phases, int only = -1,
                         bool finalize = true, const StepHdr* hin = nullptr,
                         std::vector<pk_pack::Node>* rec = nullptr) {
  cudaStream_t s = p->ctx->stream;
  int last = -1, first = -1;
  for (int i = 0; i < (int)phases.size(); ++i)
    if (phases[i].ntiles) {
      last = i;
      if (first < 0) first = i;
    }
  for (size_t i = 0; i < phases.size(); ++i) {
    const Phase& ph = phases[i];
    if (!ph.ntiles || (only >= 0 && (int)i != only)) continue;
    pk::PhaseArgs<T> a{};
    a.mems = (const MemberDev<T>*)p->d_members;
    a.hdr = (const StepHdr*)p->d_blob;
    a.feeds = (const FeedDev<T>*)(p->d_blob + sizeof(StepHdr));
    a.tiles = ph.tiles;
    a.done = p->d_done;
    a.halt = p->d_done + 1;
    a.ring = p->d_ring;
    a.ring_stride = p->ring_stride;
    a.K = p->K;
    a.is_last = finalize && (int)i == last;
    a.prefetch = (int)i == first;
    a.first = (int)i == first;
    if (p->d_trace && &phases == &p->train) {  // train phases: [phase][cta][slot]
      size_t off = 0;
      for (size_t j = 0; j < i; ++j) off += (size_t)phases[j].ntiles * pk::kTraceSlots;
      a.trace = p->d_trace + off;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ph.ntiles);
    cfg.blockDim = dim3(ph.nt);
    cfg.dynamicSmemBytes = ph.smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    a.cs = ph.cs;
    a.stages = ph.stages;
    if (ph.ntiles <= pk::kInlineTiles) {
      a.tin = 1;
      memcpy(a.tiles_in, ph.host.data(), sizeof(Tile) * ph.ntiles);
    }
    if (p->K <= pk::kInlineMems) {
      a.min_ = 1;
      memcpy(a.mems_in, p->h_mems.data(), sizeof(pk::MemberDev<T>) * p->K);
    }
    if (p->K <= pk::kInlineFeeds && &phases == &p->train) {
      a.all_tensor = 1;
      for (int k = 0; k < p->K; ++k) {
        a.ctl_in[k] = p->members[k]->ctl;
        a.all_tensor &= (p->members[k]->m1t || p->members[k]->m1x) ? 1 : 0;
      }
    }
    a.gsize = ph.gsize;
    if (hin) {  // inline descriptor (feeds staged in p->h_feeds by the caller)
      a.nin = p->K;
      a.hdr_in = *hin;
      memcpy(a.feeds_in, p->h_feeds.data(), sizeof(FeedDev<T>) * p->K);
    }
    if (ph.cs > 1) {
      attr[1].id = cudaLaunchAttributeClusterDimension;
      attr[1].val.clusterDim.x = ph.cs;
      attr[1].val.clusterDim.y = 1;
      attr[1].val.clusterDim.z = 1;
      cfg.numAttrs = 2;
    }
    PhaseKernel<T> kern = ph.special == 1   ? pk::k_mlp1_fwd<T>
                          : ph.special == 2 ? pk::k_mlp1_bwd<T>
                          : ph.special == 3 ? pk::k_m1t_fwd<T>
                          : ph.special == 4 ? pk::k_m1t_bwd<T>
                          : ph.special == 5 ? pk::k_m1s_fwd<T>
                          : ph.special == 6 ? pk::k_m1c_fwd<T>
                          : ph.special == 7 ? pk::k_m1x_step<T>
                                            : kernel_for<T>(ph.mask);
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
    if (e != cudaSuccess) {
      p->ctx->err = std::string("launch phase: ") + cudaGetErrorString(e);
      return PK_ERR_CUDA;
    }
    if (rec) {  // capturing: remember the kernel node this launch became
      cudaStreamCaptureStatus cs;
      const cudaGraphNode_t* deps = nullptr;
      size_t nd = 0;
      e = cudaStreamGetCaptureInfo(s, &cs, nullptr, nullptr, &deps, &nd);
      if (e != cudaSuccess || nd != 1) {
        p->ctx->err = "capture: cannot identify the kernel node";
        return PK_ERR_CUDA;
      }
      pk_pack::Node nd_{};
      nd_.node = deps[0];
      nd_.args.assign(reinterpret_cast<const char*>(&a), reinterpret_cast<const char*>(&a) + sizeof(a));
      nd_.kp.func = reinterpret_cast<void*>(kern);
      nd_.kp.gridDim = cfg.gridDim;
      nd_.kp.blockDim = cfg.blockDim;
      nd_.kp.sharedMemBytes = (unsigned)cfg.dynamicSmemBytes;
      rec->push_back(std::move(nd_));
    }
  }
  return PK_OK;
}

static int launch(pk_pack* p, const std::vector<Phase>& ph, int only = -1, bool fin = true) {
  return p->ctx->dtype == PK_F64 ? launch_phases<double>(p, ph, only, fin)
                                 : launch_phases<float>(p, ph, only, fin);
}

extern "C" int pk_pack_create(pk_ctx* c, pk_member* const* members, int32_t k, pk_pack** out) {
  if (!c || !out || !members || k < 1) return arg_err(c, "pack needs at least one member");
  cudaSetDevice(c->device);
  for (int i = 0; i < k; ++i) {
    if (!members[i] || members[i]->ctx != c) return arg_err(c, "pack: member from another context");
    for (int j = 0; j < i; ++j)
      if (members[j] == members[i]) return arg_err(c, "pack: duplicate member");
  }
  if (!g_smem_max[c->dtype]) {
    cudaError_t e = c->dtype == PK_F64 ? init_smem_limit<double>(c->device, &g_smem_max[1])
                                       : init_smem_limit<float>(c->device, &g_smem_max[0]);
    CK_CTX(c, e);
  }
  for (int i = 0; i < k; ++i) {  // FWD/WGRAD/DGRAD tiles must fit regardless of shape
    const int need = c->dtype == PK_F64 ? pk::Smem<double>::FWD : pk::Smem<float>::FWD;
    if (need > g_smem_max[c->dtype]) return arg_err(c, "pack: shared memory budget too small");
  }
  auto* p = new pk_pack();
  p->ctx = c;
  p->members.assign(members, members + k);
  p->K = k;
  p->inline_desc = k <= pk::kInlineFeeds && g_plan.inline_desc;
  size_t mdsz = c->dtype == PK_F64 ? sizeof(MemberDev<double>) : sizeof(MemberDev<float>);
  std::vector<char> hm(mdsz * k);
  for (int i = 0; i < k; ++i) {
    const int tl = tail_ok(members[i], c->dtype);
    if (c->dtype == PK_F64) {
      auto d = member_dev<double>(members[i], tl);
      memcpy(hm.data() + i * mdsz, &d, mdsz);
    } else {
      auto d = member_dev<float>(members[i], tl);
      memcpy(hm.data() + i * mdsz, &d, mdsz);
    }
  }
  p->h_mems = hm;
  build_phases(p, false, p->train);
  build_phases(p, true, p->eval);
  std::vector<Tile> all;
  for (auto* v : {&p->train, &p->eval})
    for (auto& ph : *v) all.insert(all.end(), ph.host.begin(), ph.host.end());
  p->blob_bytes = sizeof(StepHdr) + feed_size(c->dtype) * k;
  p->ring_stride = (int32_t)align_up(16 + 8 * (size_t)k, 64);
  auto fail = [&](cudaError_t e) {
    c->err = std::string("pack alloc: ") + cudaGetErrorString(e);
    ctx_release(c, 0, p->d_members, p->cap_members);
    ctx_release(c, 0, p->d_blob, p->cap_blob);
    ctx_release(c, 0, p->d_tiles, p->cap_tiles);
    ctx_release(c, 0, p->d_done, p->cap_done);
    ctx_release(c, 1, p->h_desc, p->cap_desc);
    ctx_release(c, 2, p->h_ring, p->cap_ring);
    delete p;
    return e == cudaErrorMemoryAllocation ? PK_ERR_OOM : PK_ERR_CUDA;
  };
  cudaError_t e;
  if ((e = ctx_alloc(c, 0, hm.size(), &p->d_members, &p->cap_members)) != cudaSuccess) return fail(e);
  if ((e = ctx_alloc(c, 0, p->blob_bytes, (void**)&p->d_blob, &p->cap_blob)) != cudaSuccess)
    return fail(e);
  // d_done: [done, halt, -, -] + the FWD split workspace (one arrival counter
  // per CTA, then kFwdMaxRanges range tiles per CTA) for the largest phase in
  // which FWD tiles are shared by several CTAs
  size_t ws_ctas = 0;
  for (auto* v : {&p->train, &p->eval})
    for (auto& ph : *v) {
      if (ph.special) continue;
      for (const Tile& t : ph.host)
        if (t.kind == pk::TK_FWD && (t.m0 >> 24)) {
          ws_ctas = std::max(ws_ctas, (size_t)ph.ntiles);
          break;
        }
    }
  const size_t es = c->dtype == PK_F64 ? 8 : 4;
  p->done_bytes = 16 + (ws_ctas ? 4 * ((ws_ctas + 3) & ~(size_t)3) +
                                      ws_ctas * pk::kFwdMaxRanges * pk::FWD_BM * pk::FWD_BN * es
                                : 0);
  if ((e = ctx_alloc(c, 0, p->done_bytes, (void**)&p->d_done, &p->cap_done)) != cudaSuccess)
    return fail(e);
  if ((e = ctx_alloc(c, 0, std::max<size_t>(1, all.size()) * sizeof(Tile), (void**)&p->d_tiles,
                     &p->cap_tiles)) != cudaSuccess)
    return fail(e);
  if ((e = ctx_alloc(c, 1, p->blob_bytes * kRing, (void**)&p->h_desc, &p->cap_desc)) != cudaSuccess)
    return fail(e);
  if ((e = ctx_alloc(c, 2, (size_t)p->ring_stride * kRing, (void**)&p->h_ring, &p->cap_ring)) !=
      cudaSuccess)
    return fail(e);
  if ((e = cudaHostGetDevicePointer((void**)&p->d_ring, p->h_ring, 0)) != cudaSuccess) return fail(e);
  memset(p->h_ring, 0, (size_t)p->ring_stride * kRing);
  cudaMemsetAsync(p->d_done, 0, p->done_bytes, c->stream);
  cudaMemcpyAsync(p->d_members, hm.data(), hm.size(), cudaMemcpyHostToDevice, c->stream);
  if (!all.empty())
    cudaMemcpyAsync(p->d_tiles, all.data(), all.size() * sizeof(Tile), cudaMemcpyHostToDevice, c->stream);
  size_t off = 0;
  for (auto* v : {&p->train, &p->eval})
    for (auto& ph : *v) {
      ph.tiles = p->d_tiles + off;
      off += ph.host.size();
    }
  for (int i = 0; i < kRing; ++i) {
    p->ev[i] = ctx_event(c);
    p->ev_pending[i] = false;
  }
  if (g_plan.trace) {
    for (auto& ph : p->train) p->trace_len += (size_t)ph.ntiles * pk::kTraceSlots;
    if ((e = cudaMalloc((void**)&p->d_trace, p->trace_len * 8)) != cudaSuccess) return fail(e);
    cudaMemsetAsync(p->d_trace, 0, p->trace_len * 8, c->stream);
  }
  if ((e = cudaStreamSynchronize(c->stream)) != cudaSuccess) return fail(e);
  c->bytes += hm.size() + p->blob_bytes + all.size() * sizeof(Tile);
  *out = p;
  return PK_OK;
}

extern "C" int64_t pk_pack_trace(pk_pack* p, uint64_t* out, int64_t cap) {
  if (!p || !p->d_trace) return -1;
  cudaSetDevice(p->ctx->device);
  if (cudaStreamSynchronize(p->ctx->stream) != cudaSuccess) return -1;
  const int64_t n = std::min<int64_t>(cap, (int64_t)p->trace_len);
  if (out && n > 0 && cudaMemcpy(out, p->d_trace, n * 8, cudaMemcpyDeviceToHost) != cudaSuccess)
    return -1;
  return (int64_t)p->trace_len;
}

extern "C" int pk_pack_destroy(pk_pack* p) {
  if (!p) return PK_ERR_ARG;
  pk_ctx* c = p->ctx;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  if (p->exec) cudaGraphExecDestroy(p->exec);
  if (p->graph) cudaGraphDestroy(p->graph);
  if (p->exec_multi) cudaGraphExecDestroy(p->exec_multi);
  if (p->graph_multi) cudaGraphDestroy(p->graph_multi);
  for (int i = 0; i < kRing; ++i) c->events.push_back(p->ev[i]);
  ctx_release(c, 0, p->d_members, p->cap_members);
  ctx_release(c, 0, p->d_blob, p->cap_blob);
  ctx_release(c, 0, p->d_tiles, p->cap_tiles);
  ctx_release(c, 0, p->d_done, p->cap_done);
  if (p->d_trace) cudaFree(p->d_trace);
  if (p->copy_stream) cudaStreamDestroy(p->copy_stream);
  for (auto& e : p->ev_copy)
    if (e) cudaEventDestroy(e);
  for (auto& s : p->run_stage) {
    if (s.d) pk_dataset_destroy(s.d);
    if (s.hx) cudaFreeHost(s.hx);
    if (s.hy) cudaFreeHost(s.hy);
  }
  ctx_release(c, 1, p->h_desc, p->cap_desc);
  ctx_release(c, 2, p->h_ring, p->cap_ring);
  delete p;
  return PK_OK;
}

extern "C" int32_t pk_pack_launches_per_step(const pk_pack* p) {
  if (!p) return -1;
  int n = 0;
  for (auto& ph : p->train) n += ph.ntiles > 0;
  return n;
}

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
  if (p->halt_dirty) {  // steps enqueued behind the failure have been skipped
    CK_CTX(c, cudaMemsetAsync(p->d_done + 1, 0, 4, c->stream));
    p->halt_dirty = false;
  }
  if (p->inline_desc) {
    // feeds + header ride in the kernel parameters of the graph's nodes
    p->h_feeds.resize(feed_size(c->dtype) * p->K);
    rc = c->dtype == PK_F64 ? fill_feeds<double>(p, feeds, p->h_feeds.data())
                            : fill_feeds<float>(p, feeds, p->h_feeds.data());
    if (rc) return rc;
    const StepHdr hdr{p->K, slot, 0, 0};
    if (!p->exec) {
      CK_CTX(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
      p->nodes.clear();
      rc = c->dtype == PK_F64 ? launch_phases<double>(p, p->train, -1, true, &hdr, &p->nodes)
                              : launch_phases<float>(p, p->train, -1, true, &hdr, &p->nodes);
      cudaError_t e = cudaStreamEndCapture(c->stream, &p->graph);
      if (rc) return rc;
      CK_CTX(c, e);
      CK_CTX(c, cudaGraphInstantiate(&p->exec, p->graph, 0));
    } else {
      const size_t o_hdr = c->dtype == PK_F64 ? offsetof(pk::PhaseArgs<double>, hdr_in)
                                              : offsetof(pk::PhaseArgs<float>, hdr_in);
      const size_t o_feeds = c->dtype == PK_F64 ? offsetof(pk::PhaseArgs<double>, feeds_in)
                                                : offsetof(pk::PhaseArgs<float>, feeds_in);
      for (auto& n : p->nodes) {
        memcpy(n.args.data() + o_hdr, &hdr, sizeof(hdr));
        memcpy(n.args.data() + o_feeds, p->h_feeds.data(), p->h_feeds.size());
        void* args[1] = {n.args.data()};
        n.kp.kernelParams = args;
        n.kp.extra = nullptr;
        CK_CTX(c, cudaGraphExecKernelNodeSetParams(p->exec, n.node, &n.kp));
      }
    }
  } else {
    if ((rc = launch_desc(p, slot, 0, feeds))) return rc;
    if (!p->exec) {
      CK_CTX(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
      rc = launch(p, p->train);
      cudaError_t e = cudaStreamEndCapture(c->stream, &p->graph);
      if (rc) return rc;
      CK_CTX(c, e);
      CK_CTX(c, cudaGraphInstantiate(&p->exec, p->graph, 0));
    }
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
  if (s[0] != PK_OK) p->halt_dirty = true;  // cleared before the next launch
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
  for (auto* m : p->members)
    max_chunks = std::max<int64_t>(max_chunks, (rows + m->desc.max_rows - 1) / m->desc.max_rows);
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
    if ((rc = launch(p, p->eval))) return rc;
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
  std::vector<int> idx;
  for (int i = 0; i < (int)p->train.size(); ++i)
    if (p->train[i].ntiles) idx.push_back(i);
  const int n = (int)idx.size();
  std::vector<cudaEvent_t> ev(n + 1);
  for (auto& e : ev) CK_CTX(c, cudaEventCreate(&e));
  // phases launched one at a time (no PDL overlap) so each is timed alone;
  // the last one keeps is_last so FINALIZE commits the step
  for (int j = 0; j < n; ++j) {
    CK_CTX(c, cudaEventRecord(ev[j], c->stream));
    if ((rc = launch(p, p->train, idx[j], j + 1 == n))) return rc;
  }
  CK_CTX(c, cudaEventRecord(ev[n], c->stream));
  CK_CTX(c, cudaEventSynchronize(ev[n]));
  for (int j = 0; j < n; ++j) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev[j], ev[j + 1]);
    const Phase& ph = p->train[idx[j]];
    if (phase_ms) phase_ms[j] = ms;
    // special (fused / tensor-path) kernels report 16 + their id
    if (phase_kind) phase_kind[j] = ph.special ? 16 + ph.special : ph.kind;
    if (phase_layer) phase_layer[j] = ph.layer;
    if (phase_ctas) phase_ctas[j] = ph.ntiles;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return read_result(p, slot, losses, st);
}


extern "C" int pk_plan_options_get(pk_plan_options* out) {
  if (!out) return PK_ERR_ARG;
  *out = g_plan;
  return PK_OK;
}

extern "C" int pk_plan_options_set(const pk_plan_options* in) {
  if (!in) {
    g_plan = plan_defaults();
    return PK_OK;
  }
  if (in->fwd < 0 || in->fwd > 2 || in->fwd_cluster < 0 || in->run_batch < 0) return PK_ERR_ARG;
  g_plan = *in;
  return PK_OK;
}
