// pk_run.cuh — native multi-step driver (included by pk_runtime.cu after
// pk_pack.cuh): `pk_pack_run` is the reference's packed_step loop
// (packing.py:185-264) planned and applied in C++, with up to `depth` steps in
// flight.  Per step it does exactly what the Python planner does:
//
//   active     members with steps_done < target_steps (shadow cursors)
//   roll       pos >= n → epoch + 1, pos 0 (packing.py:175-182)
//   groups     (dataset, epoch, pos, batch) in sorted order (packing.py:121-128)
//   rows       take = min(batch, n - pos), idx = perm_epoch[pos : pos + take]
//              (data.py:124-136); labels checked against every member's classes
//   inputs     device-resident: feed = (dataset, device order, pos, take);
//              streamed: rows gathered into a pinned slot + async H2D
//   apply      at result time, in step order: roll, then steps_done += 1,
//              pos += take, samples_used[idx] += 1 (packing.py:255-257); a
//              non-finite value commits nothing, a non-finite gradient at
//              member k commits the members before k (packing.py:246-253)
//
// The host's share of a step drops to a few microseconds, so the pipeline is
// bound by the device.  Anything the loop cannot decide alone (a permutation
// it was not given, a label out of bounds) stops it cleanly before that step
// is enqueued; the Python caller resolves it and calls again.

#pragma once

namespace {

struct RunKey {
  int32_t ds;
  int64_t epoch, pos;
  int32_t batch;
  bool operator<(const RunKey& o) const {
    if (ds != o.ds) return ds < o.ds;
    if (epoch != o.epoch) return epoch < o.epoch;
    if (pos != o.pos) return pos < o.pos;
    return batch < o.batch;
  }
  bool operator==(const RunKey& o) const {
    return ds == o.ds && epoch == o.epoch && pos == o.pos && batch == o.batch;
  }
};

struct RunStep {
  int64_t ticket;
  std::vector<int32_t> member;  // active members (pack order)
  std::vector<int32_t> take;    // rows each took
  std::vector<const int64_t*> idx;
  int32_t groups, physical, driver;
};

}  // namespace

static pk_pack::RunStage* run_stage(pk_pack* p, int slot, int gi, int64_t rows, int32_t dim) {
  auto& v = p->run_stage;
  const size_t i = (size_t)slot * p->K + gi;
  if (v.size() <= i) v.resize(i + 1);
  pk_pack::RunStage& s = v[i];
  if (s.d && (s.d->n < rows || s.d->dim != dim)) {
    pk_dataset_destroy(s.d);
    cudaFreeHost(s.hx);
    cudaFreeHost(s.hy);
    s = pk_pack::RunStage{};
  }
  if (!s.d) {
    if (pk_dataset_create(p->ctx, rows, dim, &s.d) != PK_OK) return nullptr;
    if (cudaHostAlloc(&s.hx, (size_t)rows * dim * p->ctx->esize(), cudaHostAllocDefault) !=
            cudaSuccess ||
        cudaHostAlloc((void**)&s.hy, (size_t)rows * 4, cudaHostAllocDefault) != cudaSuccess)
      return nullptr;
  }
  return &s;
}

// rows idx of a host dataset → the slot's pinned staging → H2D on the copy
// stream; the pack stream waits for that copy before the step's kernels
template <typename T>
__global__ void k_gather_rows(const T* __restrict__ src, int64_t ld,
                              const int32_t* __restrict__ src_y, const int32_t* __restrict__ perm,
                              int64_t pos, int dim, T* __restrict__ dst, int32_t* __restrict__ dst_y);

template <typename T>
static void pk_k_gather_launch(pk_pack* p, const pk_run_dataset& d, int64_t take, int64_t pos,
                               int64_t e, pk_pack::RunStage* g) {
  k_gather_rows<T><<<(unsigned)take, 128, 0, p->copy_stream>>>(
      static_cast<const T*>(d.mapped_x), d.host_ld, d.mapped_y, d.order[e]->perm, pos, d.dim,
      static_cast<T*>(g->d->feat), g->d->labels);
}

// streamed rows gathered by the GPU itself: row perm[pos + r] of the
// host-mapped dataset (read over PCIe) → staging row r; one CTA per row,
// 16-byte reads (zero-copy H2D of exactly the batch's bytes)
template <typename T>
__global__ void k_gather_rows(const T* __restrict__ src, int64_t ld,
                              const int32_t* __restrict__ src_y, const int32_t* __restrict__ perm,
                              int64_t pos, int dim, T* __restrict__ dst, int32_t* __restrict__ dst_y) {
  const int r = blockIdx.x;
  const int64_t row = perm[pos + r];
  const T* s = src + row * ld;
  T* d = dst + (int64_t)r * dim;
  constexpr int V = 16 / (int)sizeof(T);
  if ((ld % V) == 0 && (dim % V) == 0 && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
    for (int i = threadIdx.x; i < dim / V; i += blockDim.x)
      reinterpret_cast<float4*>(d)[i] = reinterpret_cast<const float4*>(s)[i];
  } else {
    for (int i = threadIdx.x; i < dim; i += blockDim.x) d[i] = s[i];
  }
  if (threadIdx.x == 0) dst_y[r] = src_y[row];
}

static int run_gather(pk_pack* p, int slot, pk_pack::RunStage* g, int64_t take,
                      const pk_run_dataset& d, const int64_t* idx, int64_t pos, int64_t e) {
  pk_ctx* c = p->ctx;
  if (!p->copy_stream) CK_CTX(c, cudaStreamCreateWithFlags(&p->copy_stream, cudaStreamNonBlocking));
  if (!p->ev_copy[slot]) CK_CTX(c, cudaEventCreateWithFlags(&p->ev_copy[slot], cudaEventDisableTiming));
  const size_t es = c->esize(), rb = (size_t)d.dim * es;
  if (d.mapped_x && d.mapped_y && d.order && d.order[e]) {
    // zero-copy: the GPU pulls the batch's rows from page-locked host memory
    if (c->dtype == PK_F64)
      pk_k_gather_launch<double>(p, d, take, pos, e, g);
    else
      pk_k_gather_launch<float>(p, d, take, pos, e, g);
    CK_CTX(c, cudaGetLastError());
  } else {
    for (int64_t i = 0; i < take; ++i) {
      memcpy((char*)g->hx + (size_t)i * rb, (const char*)d.host_x + (size_t)idx[i] * d.host_ld * es, rb);
      g->hy[i] = d.host_y[idx[i]];
    }
    CK_CTX(c, cudaMemcpyAsync(g->d->feat, g->hx, (size_t)take * rb, cudaMemcpyHostToDevice,
                              p->copy_stream));
    CK_CTX(c, cudaMemcpyAsync(g->d->labels, g->hy, (size_t)take * 4, cudaMemcpyHostToDevice,
                              p->copy_stream));
  }
  CK_CTX(c, cudaEventRecord(p->ev_copy[slot], p->copy_stream));
  CK_CTX(c, cudaStreamWaitEvent(c->stream, p->ev_copy[slot], 0));
  return PK_OK;
}

// n (>= 2) whole steps in ONE graph launch: the graph-launch gap between
// consecutive steps disappears and each step's first kernel starts (PDL)
// while the previous step drains; feeds: n x K (inline descriptors only)
static int step_multi_async(pk_pack* p, const pk_feed* feeds, int n, int64_t* tickets) {
  pk_ctx* c = p->ctx;
  std::vector<int> slots(n);
  for (int s = 0; s < n; ++s) {
    int rc = acquire_slot(p, p->next_ticket + s, &slots[s]);
    if (rc) return rc;
  }
  if (p->halt_dirty) {
    CK_CTX(c, cudaMemsetAsync(p->d_done + 1, 0, 4, c->stream));
    p->halt_dirty = false;
  }
  const size_t fs = feed_size(c->dtype) * p->K;
  p->h_feeds.resize(fs);
  const bool f64 = c->dtype == PK_F64;
  if (!p->exec_multi || p->multi_n != n) {
    if (p->exec_multi) cudaGraphExecDestroy(p->exec_multi);
    if (p->graph_multi) cudaGraphDestroy(p->graph_multi);
    p->exec_multi = nullptr;
    p->graph_multi = nullptr;
    p->nodes_multi.assign(n, {});
    CK_CTX(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    int rc = PK_OK;
    for (int s = 0; s < n && rc == PK_OK; ++s) {
      rc = f64 ? fill_feeds<double>(p, feeds + (size_t)s * p->K, p->h_feeds.data())
               : fill_feeds<float>(p, feeds + (size_t)s * p->K, p->h_feeds.data());
      if (rc) break;
      const StepHdr hdr{p->K, slots[s], 0, 0};
      rc = f64 ? launch_phases<double>(p, p->train, -1, true, &hdr, &p->nodes_multi[s])
               : launch_phases<float>(p, p->train, -1, true, &hdr, &p->nodes_multi[s]);
    }
    cudaError_t e = cudaStreamEndCapture(c->stream, &p->graph_multi);
    if (rc) return rc;
    CK_CTX(c, e);
    CK_CTX(c, cudaGraphInstantiate(&p->exec_multi, p->graph_multi, 0));
    p->multi_n = n;
  } else {
    const size_t o_hdr = f64 ? offsetof(pk::PhaseArgs<double>, hdr_in)
                             : offsetof(pk::PhaseArgs<float>, hdr_in);
    const size_t o_feeds = f64 ? offsetof(pk::PhaseArgs<double>, feeds_in)
                               : offsetof(pk::PhaseArgs<float>, feeds_in);
    for (int s = 0; s < n; ++s) {
      int rc = f64 ? fill_feeds<double>(p, feeds + (size_t)s * p->K, p->h_feeds.data())
                   : fill_feeds<float>(p, feeds + (size_t)s * p->K, p->h_feeds.data());
      if (rc) return rc;
      const StepHdr hdr{p->K, slots[s], 0, 0};
      for (auto& nd : p->nodes_multi[s]) {
        memcpy(nd.args.data() + o_hdr, &hdr, sizeof(hdr));
        memcpy(nd.args.data() + o_feeds, p->h_feeds.data(), fs);
        void* args[1] = {nd.args.data()};
        nd.kp.kernelParams = args;
        nd.kp.extra = nullptr;
        CK_CTX(c, cudaGraphExecKernelNodeSetParams(p->exec_multi, nd.node, &nd.kp));
      }
    }
  }
  CK_CTX(c, cudaGraphLaunch(p->exec_multi, c->stream));
  for (int s = 0; s < n; ++s) {
    CK_CTX(c, cudaEventRecord(p->ev[slots[s]], c->stream));
    p->ev_pending[slots[s]] = true;
    tickets[s] = p->next_ticket + s;
  }
  p->next_ticket += n;
  return PK_OK;
}

static void run_roll(pk_run_member& m, const pk_run_dataset& d) {
  if (m.pos >= d.n) {
    m.epoch += 1;
    m.pos = 0;
    if (m.samples_used) memset(m.samples_used, 0, sizeof(int64_t) * (size_t)d.n);
  }
}

extern "C" int pk_pack_run(pk_pack* p, pk_run_member* mem, const pk_run_dataset* ds, int32_t n_ds,
                           int32_t share_inputs, int64_t max_steps, int32_t depth, double* losses,
                           uint8_t* active, int32_t* stats, int64_t* done, pk_status* st,
                           int32_t* stop) {
  if (!p || !mem || !ds || n_ds < 1 || !losses || !active || !stats || !done || !st || !stop)
    return PK_ERR_ARG;
  pk_ctx* c = p->ctx;
  cudaSetDevice(c->device);
  const int K = p->K;
  depth = std::max(1, std::min(depth, kRing));
  *done = 0;
  *stop = PK_RUN_MAX_STEPS;
  st->code = PK_OK;
  st->member = -1;
  st->index = -1;
  st->committed = 0;
  for (int k = 0; k < K; ++k)
    if (mem[k].dataset < 0 || mem[k].dataset >= n_ds) return arg_err(c, "run: bad dataset index");
  // shadow cursors: the state after every enqueued step commits
  std::vector<pk_run_member> sh(mem, mem + K);
  for (auto& m : sh) m.samples_used = nullptr;  // the shadow never touches bookkeeping
  std::vector<pk_feed> feeds(K);
  std::vector<RunStep> fly;  // in flight, oldest first
  size_t head = 0;
  int64_t planned = 0, applied = 0;
  bool more = true;
  int rc = PK_OK;
  // steps per graph launch (whole steps chained by PDL in one graph)
  int nb = 8;  // measured: config0 30.2 → 27.4 (4) → 26.3 µs/step (8)
  if (g_plan.run_batch > 0) nb = g_plan.run_batch;
  if (!p->inline_desc) nb = 1;
  nb = std::min(nb, depth);
  std::vector<RunStep> pend;     // planned, not yet launched
  std::vector<pk_feed> pfeeds;   // their feeds, K per step
  auto flush = [&]() -> int {
    const int n = (int)pend.size();
    if (!n) return PK_OK;
    if (n >= 2 && n == nb) {
      std::vector<int64_t> t(n);
      int r = step_multi_async(p, pfeeds.data(), n, t.data());
      if (r) return r;
      for (int i = 0; i < n; ++i) pend[i].ticket = t[i];
    } else {
      for (int i = 0; i < n; ++i) {
        int r = pk_pack_step_async(p, pfeeds.data() + (size_t)i * K, &pend[i].ticket);
        if (r) {  // the steps already launched are in flight: account for them
          for (int q = 0; q < i; ++q) fly.push_back(std::move(pend[q]));
          pend.clear();
          pfeeds.clear();
          return r;
        }
      }
    }
    for (auto& q : pend) fly.push_back(std::move(q));
    pend.clear();
    pfeeds.clear();
    return PK_OK;
  };
  // result of the oldest in-flight step → the real cursors (the reference's
  // bookkeeping); `failed`: the step hit a non-finite value / gradient, the
  // later in-flight steps were skipped on the device (halt flag)
  auto apply_oldest = [&](bool& failed) -> int {
    RunStep& s = fly[head++];
    double* L = losses + (size_t)applied * K;
    pk_status rs{};
    int r = pk_pack_step_wait(p, s.ticket, L, &rs);
    if (r != PK_OK && r != PK_ERR_NONFINITE_VALUE && r != PK_ERR_NONFINITE_GRAD) return r;
    uint8_t* A = active + (size_t)applied * K;
    memset(A, 0, K);
    if (applied > 0)  // the reference rolls at the top of every later step
      for (int k : s.member) run_roll(mem[k], ds[mem[k].dataset]);
    const bool fail = rs.code != PK_OK;
    for (size_t q = 0; q < s.member.size(); ++q) {
      const int k = s.member[q];
      if (rs.code == PK_ERR_NONFINITE_VALUE) break;
      if (rs.code == PK_ERR_NONFINITE_GRAD && k >= rs.member) continue;  // pack order
      pk_run_member& m = mem[k];
      m.steps_done += 1;
      m.pos += s.take[q];
      if (m.samples_used)
        for (int32_t r2 = 0; r2 < s.take[q]; ++r2) m.samples_used[s.idx[q][r2]] += 1;
      A[k] = 1;
    }
    stats[3 * applied] = s.groups;
    stats[3 * applied + 1] = s.physical;
    stats[3 * applied + 2] = s.driver;
    if (fail) {
      *st = rs;
      *stop = PK_RUN_FAILED;
      *done = applied;  // the failed step is reported through st, not counted
      for (size_t i = head; i < fly.size(); ++i) {  // skipped on the device (halt)
        pk_status sk{};
        pk_pack_step_wait(p, fly[i].ticket, L, &sk);
      }
      head = fly.size();
      failed = true;
      return PK_OK;
    }
    ++applied;
    *done = applied;
    return PK_OK;
  };
  // an error after steps were launched: their results still reach the cursors
  // (they commit on the device), so *done and the host state stay in step with
  // the device; then the error is returned
  auto bail = [&](int err) -> int {
    while (head < fly.size()) {
      bool failed = false;
      if (apply_oldest(failed) || failed) break;
    }
    *done = applied;
    return err;
  };
  while (applied < max_steps) {
    // ---- plan + enqueue while the window has room --------------------------
    while (more && (int)(fly.size() - head + pend.size()) < depth && planned < max_steps) {
      std::vector<int32_t> act;
      for (int k = 0; k < K; ++k)
        if (sh[k].steps_done < sh[k].target_steps) act.push_back(k);
      if (act.empty()) {
        more = false;
        *stop = PK_RUN_NO_MEMBER;
        break;
      }
      for (int k : act) run_roll(sh[k], ds[sh[k].dataset]);  // shadow roll (no bookkeeping)
      std::vector<std::pair<RunKey, int32_t>> keyed;
      int32_t driver = 0;
      for (int k : act) {
        keyed.push_back({RunKey{sh[k].dataset, sh[k].epoch, sh[k].pos, sh[k].batch}, k});
        driver = std::max(driver, sh[k].batch);
      }
      std::stable_sort(keyed.begin(), keyed.end(),
                       [](const auto& a, const auto& b) { return a.first < b.first; });
      // every group's permutation must be known and its labels in bounds
      bool ok = true;
      for (size_t i = 0; i < keyed.size() && ok; ++i) {
        const RunKey& key = keyed[i].first;
        const pk_run_dataset& d = ds[key.ds];
        const int64_t e = key.epoch - d.epoch0;
        if (e < 0 || e >= d.n_epochs || !d.perm[e]) {
          *stop = PK_RUN_NEED_PERM;
          ok = false;
          break;
        }
        const pk_member* m = p->members[keyed[i].second];
        if (d.max_label >= m->desc.dims[m->desc.n_layers]) {
          const int64_t take = std::min<int64_t>(key.batch, d.n - key.pos);
          const int64_t* idx = d.perm[e] + key.pos;
          for (int64_t r = 0; r < take; ++r)
            if (d.host_y[idx[r]] >= m->desc.dims[m->desc.n_layers]) {
              *stop = PK_RUN_LABEL_BOUNDS;
              ok = false;
              break;
            }
        }
      }
      if (!ok) {
        more = false;
        break;
      }
      RunStep s;
      s.driver = driver;
      s.groups = 0;
      s.physical = 0;
      for (int k = 0; k < K; ++k) feeds[k] = pk_feed{nullptr, nullptr, 0, 0, 0};
      const int slot = (int)(planned % depth);
      for (size_t i = 0; i < keyed.size();) {
        size_t j = i;
        while (j < keyed.size() && keyed[j].first == keyed[i].first) ++j;
        const RunKey& key = keyed[i].first;
        const pk_run_dataset& d = ds[key.ds];
        const int64_t* perm = d.perm[key.epoch - d.epoch0];
        const int32_t take = (int32_t)std::min<int64_t>(key.batch, d.n - key.pos);
        const int gi = s.groups;
        pk_feed f{};
        if (d.host_x) {  // streamed: gather into this slot's pinned staging, H2D
          pk_pack::RunStage* g = run_stage(p, slot, gi, std::max<int64_t>(take, driver), d.dim);
          if (!g) return bail(arg_err(c, "run: staging allocation failed"));
          if ((rc = run_gather(p, slot, g, take, d, perm + key.pos, key.pos,
                               key.epoch - d.epoch0)))
            return bail(rc);
          f = pk_feed{g->d, nullptr, 0, take, gi};
        } else {
          const int64_t e = key.epoch - d.epoch0;
          if (!d.device || !d.order || !d.order[e])
            return bail(arg_err(c, "run: missing device order"));
          f = pk_feed{d.device, d.order[e], key.pos, take, gi};
        }
        for (size_t q = i; q < j; ++q) {
          const int k = keyed[q].second;
          feeds[k] = f;
          s.member.push_back(k);
          s.take.push_back(take);
          s.idx.push_back(perm + key.pos);
        }
        s.physical += share_inputs ? 1 : (int32_t)(j - i);
        ++s.groups;
        i = j;
      }
      for (size_t q = 0; q < s.member.size(); ++q) {
        pk_run_member& m = sh[s.member[q]];
        m.steps_done += 1;
        m.pos += s.take[q];
      }
      pfeeds.insert(pfeeds.end(), feeds.begin(), feeds.end());
      pend.push_back(std::move(s));
      ++planned;
      if ((int)pend.size() == nb && (rc = flush())) return bail(rc);
    }
    // a partial batch launches when nothing more can be planned (or nothing
    // older is left to wait for)
    if (!pend.empty() && (!more || planned >= max_steps || fly.size() == head))
      if ((rc = flush())) return bail(rc);
    if (fly.size() == head) break;
    // ---- oldest step: result → the real cursors ------------------------------
    bool failed = false;
    if ((rc = apply_oldest(failed))) return bail(rc);
    if (failed) return PK_OK;
  }
  *done = applied;
  return PK_OK;
}
