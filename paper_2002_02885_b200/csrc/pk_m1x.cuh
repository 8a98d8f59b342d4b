// pk_m1x.cuh — the whole one-hidden-layer packed step in ONE launch
// (included by pk_kernels.cuh after pk_m1t.cuh).
//
// One thread-block cluster per member; cluster rank q owns hidden units
// [q·U, (q+1)·U), U = 16·bpc, and keeps them for the whole step:
//
//   forward   Z0/A0[:, units] = act(X·W0[:, units] + b0)   (FFMA, X rows
//             gathered through the epoch order, X / W0 chunks streamed by a
//             cp.async ring)
//             P_b = A0[:, block b]·W1[block b, :]  for each own 16-unit block
//   exchange  cluster barrier; every CTA sums all blocks' P_b over DSMEM in
//             block order (+ b1) → the same logits everywhere → softmax-xent
//             → dZ1 (rank 0 writes the loss terms)
//   backward  dZ0[:, units] = (dZ1·W1[units, :]ᵀ) ⊙ act'(Z0);
//             W1[units, :], b0[units] (+ b1 on rank 0) updated in place;
//             dW0 = Xᵀ·dZ0 chunk by chunk, consumed at once by the optimizer
//             against W0 / slot chunks staged in the same ring → Pn / Sn
//
// Nothing but the loss terms and the updated parameters reaches global
// memory: no Z/A/logit round trips, no second launch.  Packs of latency-
// bound members (batch <= 64) take this path; larger batches the tcgen05
// path (pk_m1t.cuh).
//
// Arithmetic order depends only on the member's own shape, never on U (the
// cluster size a pack picks), on K or on the other members:
//   Z0[r,u]   input quads k/4 ≡ s (mod 8) accumulate alone (k ascending) into
//             p_s; z = ((p0+p1)+(p2+p3)) + ((p4+p5)+(p6+p7)) + b0[u]
//   logits    Σ_b P_b in block order, P_b = Σ_{j<16} (j ascending), + b1
//   dW0[d,u]  rows in groups of 8 (r ascending), groups folded by the same
//             fixed pairwise tree
// so packed == standalone bit for bit (tests/test_pack.py:57-82).
//
// (included inside namespace pk)

constexpr int X_KC = 64;         // input dims per streamed chunk
constexpr int X_LD = X_KC + 4;   // X chunk row stride: 8 consecutive rows' LDS.128 are conflict-free
constexpr int X_UB = 16;         // hidden units per partial-logit block
constexpr int X_FS = 4;          // forward chunk stages
constexpr int X_RED = 4096;      // fold buffer (floats): 8/NI partial sets of RP·U
constexpr int X_MAXC = 32;       // classes on this path
constexpr int X_MAXR = 64;       // rows on this path
constexpr int X_MAXCS = 16;      // cluster size (non-portable)

__host__ __device__ inline int x_nblk(int H) { return (H + X_UB - 1) / X_UB; }
__host__ __device__ inline int x_r4(int n) { return (n + 3) & ~3; }
// largest blocks per CTA the register tiling allows: RP·U <= 2048
__host__ __device__ inline int x_bpc_max(int RP) { return RP <= 32 ? 4 : 2; }

struct M1X {
  // W0 / slot chunk rows are U + 4 floats: the optimizer pass reads 16
  // consecutive rows per warp without bank conflicts
  __host__ __device__ static int wld(int U) { return U + 4; }
  __host__ __device__ static int fwd_stage(int RP, int U) { return RP * X_LD + X_KC * wld(U); }
  __host__ __device__ static int bwd_stage(int RP, int U, int ns) {
    return RP * X_LD + (1 + ns) * X_KC * wld(U);
  }
  __host__ __device__ static int ring(int RP, int U, int ns, int Sb) {
    const int a = X_FS * fwd_stage(RP, U), b = Sb * bwd_stage(RP, U, ns);
    return a > b ? a : b;
  }
  // dynamic smem bytes of one CTA (U = 16·bpc units, Sb backward stages)
  __host__ __device__ static int smem(int RP, int U, int C, int ns, int Sb) {
    return 4 * (ring(RP, U, ns, Sb) + X_RED + 3 * RP * U + x_r4(U * C) +
                x_r4((U / X_UB) * RP * C) + x_r4(RP * (C + 1)) + x_r4(U) + 32) +
           8 * RP;
  }
};

// a[4i + j] += Σ_k x[i].k · w[k].j, k ascending
__device__ __forceinline__ void x_fma4x4(float (&a)[16], const float4 (&x)[4], const float4 (&w)[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float xs[4] = {x[i].x, x[i].y, x[i].z, x[i].w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float ws[4] = {w[k].x, w[k].y, w[k].z, w[k].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) a[4 * i + j] = fmaf(xs[k], ws[j], a[4 * i + j]);
    }
  }
}

// fold the NI (1, 2, 4) consecutive partials one thread holds: fixed pairwise tree
template <int NI>
__device__ __forceinline__ float x_fold(const float (&acc)[NI][16], int e) {
  if constexpr (NI == 1) return acc[0][e];
  else if constexpr (NI == 2) return acc[0][e] + acc[1][e];
  else return (acc[0][e] + acc[1][e]) + (acc[2][e] + acc[3][e]);
}

// finish the same tree over G (1, 2, 4, 8) stored partials p[0], p[st], ...
template <int G, typename V>
__device__ __forceinline__ V x_tree(const V* p, int st) {
  auto add = [](V a, V b) {
    if constexpr (sizeof(V) == 4) return a + b;
    else return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
  };
  if constexpr (G == 1) return p[0];
  else if constexpr (G == 2) return add(p[0], p[st]);
  else if constexpr (G == 4) return add(add(p[0], p[st]), add(p[2 * st], p[3 * st]));
  else
    return add(add(add(p[0], p[st]), add(p[2 * st], p[3 * st])),
               add(add(p[4 * st], p[5 * st]), add(p[6 * st], p[7 * st])));
}

template <int RP, int BPC>
__device__ __forceinline__ void m1x_step_t(char* sm, const MemberDev<float>& M,
                                           const FeedDev<float>& f, int q, int Sb) {
  const int OPT = M.opt, NS = M.n_slots;
  constexpr int U = X_UB * BPC, WLD = U + 4, CW = U / 4;
  constexpr int NI = RP * U / 512;           // work items per thread: 1, 2, 4
  constexpr int RQ = RP / 4, CELLS = RP * U / 16, G8 = 8 / NI;
  constexpr int GB = (RP / 8) / NI;          // stored 8-row-group partials (backward)
  static_assert(NI == 1 || NI == 2 || NI == 4, "RP * U must be 512, 1024 or 2048");
  const int D = M.dims[0], H = M.dims[1], C = M.dims[2];
  const int R = f.take;
  const int ns = NS;
  const int u0 = q * U;
  const int nu = max(0, min(U, H - u0));  // own valid units (H % 4 == 0: whole quads)
  const int nblk = x_nblk(H);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const MemberCtl* ctl = M.ctl;
  const int64_t NP = M.s_stride;
  const bool work = nu > 0;  // CTA-uniform: a rank past H only joins the barriers
  // the batch's gather index first: its cold load flies with the parity load
  int myrow = 0;
  if (tid < R) myrow = (int32_t)feed_row(f, tid);
  const int par = ctl->parity;
  const float* __restrict__ Pc = M.params[par];
  float* __restrict__ Pn = M.params[par ^ 1];
  const float* __restrict__ Sc = M.slots[par];
  float* __restrict__ Sn = M.slots[par ^ 1];
  // ---- shared memory carve ----------------------------------------------------
  const int SF = M1X::fwd_stage(RP, U), SB = M1X::bwd_stage(RP, U, ns);
  float* ring = reinterpret_cast<float*>(sm);
  float* sRed = ring + M1X::ring(RP, U, ns, Sb);
  float* sZ = sRed + X_RED;                 // [RP][U] Z0 of own units
  float* sA = sZ + RP * U;                  // [RP][U] A0
  float* sdZ = sA + RP * U;                 // [RP][U] dZ0
  float* sW1 = sdZ + RP * U;                // [U][C] W1 rows of own units (zero past H)
  float* sPL = sW1 + x_r4(U * C);           // [BPC][RP][C] own blocks' partial logits
  float* sL = sPL + x_r4(BPC * RP * C);     // [RP][C+1] logits → dZ1
  float* sb0 = sL + x_r4(RP * (C + 1));     // [U]
  float* sb1 = sb0 + x_r4(U);               // [32]
  int32_t* srow = reinterpret_cast<int32_t*>(sb1 + 32);
  int32_t* ylab = srow + RP;
  const int LDL = C + 1;
  const int nch = (D + X_KC - 1) / X_KC;
  const int64_t w0 = M.w_off[0], w1 = M.w_off[1];

  // ---- prologue ----------------------------------------------------------------
  // refill addressing, fixed per thread for the whole step: X items (row r,
  // quad j) and W items (chunk row k, unit quad j)
  constexpr int XI = RP * (X_KC / 4) / NT, WI = X_KC * CW / NT > 0 ? X_KC * CW / NT : 1;
  static_assert(RP * (X_KC / 4) % NT == 0, "X refill items");
  int wk[WI], wj[WI];
#pragma unroll
  for (int i = 0; i < WI; ++i) {
    const int e = tid + NT * i;
    wk[i] = e / CW;
    wj[i] = e % CW;
  }
  auto issue_w = [&](int c, float* W, const float* src) {  // rows of a [D][H] block, own units
    const int k0 = c * X_KC;
#pragma unroll
    for (int i = 0; i < WI; ++i) {
      if (tid + NT * i >= X_KC * CW) break;
      const bool ok = k0 + wk[i] < D && 4 * wj[i] < nu;
      cp_async<16>(W + wk[i] * WLD + 4 * wj[i],
                   ok ? src + (int64_t)(k0 + wk[i]) * H + u0 + 4 * wj[i] : Pc, ok);
    }
  };
  const float* xsrc[XI];  // row bases (set once the gather index is in smem)
  int xr[XI], xj[XI];
  auto issue_x = [&](int c, float* X) {
    const int k0 = c * X_KC;
#pragma unroll
    for (int i = 0; i < XI; ++i) {
      const bool ok = xr[i] < R && k0 + 4 * xj[i] < D;
      cp_async<16>(X + xr[i] * X_LD + 4 * xj[i], ok ? xsrc[i] + k0 : f.feat, ok);
    }
  };
  // group 0: W1 rows / b0 slice / b1 and the first X_FS W0 chunks of own units
  if (work) {
    for (int e = tid; e < (nu * C) / 4; e += NT)
      cp_async<16>(sW1 + 4 * e, Pc + w1 + (int64_t)u0 * C + 4 * e, true);
    for (int e = nu * C + tid; e < U * C; e += NT) sW1[e] = 0.f;
    for (int e = tid; e < CW; e += NT)
      cp_async<16>(sb0 + 4 * e, 4 * e < nu ? Pc + M.b_off[0] + u0 + 4 * e : Pc, 4 * e < nu);
    for (int c = tid; c < C; c += NT) cp_async<4>(sb1 + c, Pc + M.b_off[1] + c, true);
    for (int c = 0; c < X_FS && c < nch; ++c) issue_w(c, ring + c * SF + RP * X_LD, Pc + w0);
    // the backward's optimizer slots (cold HBM) toward L2 now: one plain
    // prefetch per row segment (bulk prefetches would queue in the TMA unit)
    for (int e = tid; e < NS * D; e += NT) {
      const int s = e / D, k = e % D;
      const float* a = Sc + (int64_t)s * NP + w0 + (int64_t)k * H + u0;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
      if (U > 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(a + 32));
    }
  }
  cp_commit();
  if (tid < RP) srow[tid] = myrow;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < XI; ++i) {
    const int e = tid + NT * i;
    xr[i] = e / (X_KC / 4);
    xj[i] = e % (X_KC / 4);
    xsrc[i] = f.feat + (int64_t)srow[xr[i]] * f.ld + 4 * xj[i];
  }
  // labels: needed at the softmax only — the load flies through the forward
  const int mylab = tid < R ? f.labels[myrow] : 0;
  int issued = 0;  // chunk commit groups issued so far
  if (work)
    for (int c = 0; c < X_FS && c < nch; ++c) {
      issue_x(c, ring + c * SF);
      cp_commit();
      ++issued;
    }
  PK_TRACE(1);

  // ---- forward: Z0 partials ---------------------------------------------------
  // thread = (4-row x 4-unit cell, subset group): subsets grp·NI + [0, NI)
  const int cell = tid % CELLS, grp = tid / CELLS;
  const int rq = cell % RQ, uq = cell / RQ;  // rows rq + RQ·i, units 4uq..4uq+3
  float acc[NI][16];
#pragma unroll
  for (int i = 0; i < NI; ++i)
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[i][e] = 0.f;
  if (work) {
    const int nfull = D / X_KC;  // chunks without a ragged tail
    for (int c = 0; c < nch; ++c) {
      cp_wait_n(issued - c - 1);
      __syncthreads();  // chunk c landed everywhere; chunk c-1's stage is free
      if (c - 1 + X_FS < nch && c >= 1) {
        float* st = ring + ((c - 1) % X_FS) * SF;
        issue_x(c - 1 + X_FS, st);
        issue_w(c - 1 + X_FS, st + RP * X_LD, Pc + w0);
        cp_commit();
        ++issued;
      }
      const float* X = ring + (c % X_FS) * SF + rq * X_LD;
      const float* W = ring + (c % X_FS) * SF + RP * X_LD + 4 * uq;
      if (c < nfull) {
        // 2·NI quads per thread; the next quad's operands load while the
        // current one multiplies
        float4 xv[2][4], wv[2][4];
        auto ld = [&](int t, float4 (&x)[4], float4 (&w)[4]) {
          const int qi = 8 * (t / NI) + grp * NI + t % NI;  // subset qi % 8
#pragma unroll
          for (int i = 0; i < 4; ++i) x[i] = *reinterpret_cast<const float4*>(X + RQ * i * X_LD + 4 * qi);
#pragma unroll
          for (int k = 0; k < 4; ++k) w[k] = *reinterpret_cast<const float4*>(W + (4 * qi + k) * WLD);
        };
        ld(0, xv[0], wv[0]);
#pragma unroll
        for (int t = 0; t < 2 * NI; ++t) {
          if (t + 1 < 2 * NI) ld(t + 1, xv[(t + 1) & 1], wv[(t + 1) & 1]);
          x_fma4x4(acc[t % NI], xv[t & 1], wv[t & 1]);
        }
      } else {
        const int nq = (D - c * X_KC) / 4;
#pragma unroll
        for (int t = 0; t < 2 * NI; ++t) {
          const int qi = 8 * (t / NI) + grp * NI + t % NI;
          if (qi < nq) {
            float4 xv[4], wv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) xv[i] = *reinterpret_cast<const float4*>(X + RQ * i * X_LD + 4 * qi);
#pragma unroll
            for (int k = 0; k < 4; ++k) wv[k] = *reinterpret_cast<const float4*>(W + (4 * qi + k) * WLD);
            x_fma4x4(acc[t % NI], xv, wv);
          }
        }
      }
    }
    // this thread's subsets, pre-folded, → sRed[grp][r][u]
#pragma unroll
    for (int i = 0; i < 4; ++i)
      *reinterpret_cast<float4*>(sRed + (grp * RP + rq + RQ * i) * U + 4 * uq) =
          make_float4(x_fold<NI>(acc, 4 * i), x_fold<NI>(acc, 4 * i + 1),
                      x_fold<NI>(acc, 4 * i + 2), x_fold<NI>(acc, 4 * i + 3));
  }
  __syncthreads();  // ring free: the backward's first chunks fly during the exchange
  int issued_b = 0;
  auto issue_b = [&](int c) {
    float* st = ring + (c % Sb) * SB;
    issue_x(c, st);
    for (int s = 0; s <= ns; ++s)
      issue_w(c, st + RP * X_LD + s * X_KC * WLD, (s == 0 ? Pc : Sc + (int64_t)(s - 1) * NP) + w0);
    cp_commit();
    ++issued_b;
  };
  if (work)
    for (int c = 0; c < Sb && c < nch; ++c) issue_b(c);
  if (tid < RP) ylab[tid] = mylab;
  PK_TRACE(2);
  // ---- Z0 = tree(partials) + b0, A0 = act(Z0) ---------------------------------
  int bad = INT_MAX;
  if (work)
    for (int e = tid; e < RP * U; e += NT) {
      const int r = e / U, u = e % U;
      const bool ok = r < R && u < nu;
      const float z = x_tree<G8>(sRed + e, RP * U) + sb0[u];
      const float a = act_fwd(M.act, z);
      if (ok && !finite(z)) bad = min(bad, 1);
      if (ok && !finite(a)) bad = min(bad, 2);
      sZ[e] = ok ? z : 0.f;
      sA[e] = ok ? a : 0.f;
    }
  if (__syncthreads_or(bad != INT_MAX)) {
    // rare path: a non-finite Z0 anywhere in a row means a non-finite input
    // (node 0, engine.py:233-235) or a non-finite parameter (node 1/2)
    bool badx = false;
    for (int e = tid; e < R * D; e += NT) badx |= !finite(f.feat[(int64_t)srow[e / D] * f.ld + e % D]);
    badx = __syncthreads_or(badx);
    if (tid == 0) flag_min(&M.ctl->bad_node, badx ? 0 : 1);
    if (!badx && bad != INT_MAX) flag_min(&M.ctl->bad_node, bad);
  }
  // ---- own blocks' partial logits P_b[r][c] = Σ_{j<16} A0[r][16b+j]·W1[16b+j][c]
  for (int e = tid; work && e < BPC * RP * C; e += NT) {
    const int b = e / (RP * C), rc = e % (RP * C), r = rc / C, c = rc % C;
    const float* a = sA + r * U + X_UB * b;
    const float* w = sW1 + X_UB * b * C + c;
    float p = 0.f;
#pragma unroll
    for (int j = 0; j < X_UB; ++j) p = fmaf(a[j], w[j * C], p);
    sPL[e] = p;
  }
  umma::cluster_sync();  // every rank's partials are visible cluster-wide
  PK_TRACE(3);
  // ---- logits = Σ_b P_b (block order, over DSMEM) + b1 → sL --------------------
  bad = INT_MAX;
  for (int e = tid; e < R * C; e += NT) {
    const int r = e / C, c = e % C;
    const uint32_t la = umma::smem_u32(sPL + r * C + c);
    float z = 0.f;
    for (int b0 = 0; b0 < nblk; b0 += 8) {  // eight remote loads in flight
      float v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int b = b0 + j;
        v[j] = b < nblk ? umma::dsmem_ld(la + (uint32_t)((b % BPC) * RP * C * 4), (uint32_t)(b / BPC))
                        : 0.f;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (b0 + j < nblk) z = (b0 + j == 0) ? v[j] : z + v[j];
    }
    z += sb1[c];
    sL[r * LDL + c] = z;
    if (!finite(z)) bad = 3;
  }
  umma::cluster_arrive_relaxed();  // done reading peers (waited for before exit)
  if (q == 0 && bad != INT_MAX) flag_min(&M.ctl->bad_node, bad);
  __syncthreads();
  // ---- softmax-xent → dZ1 in sL (every rank; rank 0 writes the loss terms) --
  for (int r0 = 0; r0 < R; r0 += NT / 8) {
    const int r = r0 + (tid >> 3);
    xent_row8(sL + min(r, R - 1) * LDL, C, ylab[min(r, R - 1)], R, r < R,
              q == 0 && r < R ? M.rowloss + r : nullptr);
  }
  __syncthreads();
  PK_TRACE(8);
  if (q == 0 && warp == 0) {
    // the member's step loss (finalize's lane-strided order) and Adam's bias
    // corrections for the next update
    double s = 0.0;
    for (int r = lane; r < R; r += 32) s += M.rowloss[r];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      MemberCtl* c = M.ctl;
      c->loss = s / double(R);
      adam_bias_corrections(c->step_counter + 1, &c->bcn1, &c->bcn2);
    }
  }
  // ---- dZ0 = (dZ1 · W1[units, :]ᵀ) ⊙ act'(Z0, A0) -----------------------------
  if (work)
    for (int e = tid; e < RP * U; e += NT) {
      const int r = e / U, u = e % U;
      float v = 0.f;
      if (r < R && u < nu) {
        float s = 0.f;
        for (int c = 0; c < C; ++c) s = fmaf(sL[r * LDL + c], sW1[u * C + c], s);
        v = act_bwd(M.act, sZ[e], sA[e], s);
      }
      sdZ[e] = v;
    }
  __syncthreads();
  PK_TRACE(9);
  const float lr = float(ctl->lr), wd = float(M.wd);
  float bc1, bc2;  // (reciprocals)
  opt_recips(OPT, ctl, &bc1, &bc2);
  const int fault = ctl->fault_grad;
  bool badW1 = false, badb1 = false, badW0 = false, badb0 = false;
  // ---- W1[units, :] (grad 0), b1 (grad 1, rank 0), b0[units] (grad 3) --------
  for (int e = tid; e < nu * C; e += NT) {
    const int j = e / C, c = e % C;
    float g = 0.f;
    for (int r = 0; r < R; ++r) g = fmaf(sA[r * U + j], sL[r * LDL + c], g);
    if (fault == 0) g = NAN;
    badW1 |= !finite(g);
    const int64_t i = w1 + (int64_t)u0 * C + e;
    float w = sW1[e], s0 = ns >= 1 ? Sc[i] : 0.f, s1 = ns >= 2 ? Sc[NP + i] : 0.f;
    opt_step1(OPT, lr, wd, bc1, bc2, w, s0, s1, g);
    Pn[i] = w;
    if (ns >= 1) Sn[i] = s0;
    if (ns >= 2) Sn[NP + i] = s1;
  }
  if (q == 0)
    for (int c = tid; c < C; c += NT) {
      float g = 0.f;
      for (int r = 0; r < R; ++r) g += sL[r * LDL + c];
      if (fault == 1) g = NAN;
      badb1 |= !finite(g);
      const int64_t i = M.b_off[1] + c;
      float w = sb1[c], s0 = ns >= 1 ? Sc[i] : 0.f, s1 = ns >= 2 ? Sc[NP + i] : 0.f;
      opt_step1(OPT, lr, wd, bc1, bc2, w, s0, s1, g);
      Pn[i] = w;
      if (ns >= 1) Sn[i] = s0;
      if (ns >= 2) Sn[NP + i] = s1;
    }
  for (int j = tid; j < nu; j += NT) {
    float g = 0.f;
    for (int r = 0; r < R; ++r) g += sdZ[r * U + j];
    if (fault == 3) g = NAN;
    badb0 |= !finite(g);
    const int64_t i = M.b_off[0] + u0 + j;
    float w = sb0[j], s0 = ns >= 1 ? Sc[i] : 0.f, s1 = ns >= 2 ? Sc[NP + i] : 0.f;
    opt_step1(OPT, lr, wd, bc1, bc2, w, s0, s1, g);
    Pn[i] = w;
    if (ns >= 1) Sn[i] = s0;
    if (ns >= 2) Sn[NP + i] = s1;
  }
  // ---- dW0 = Xᵀ·dZ0 chunk by chunk → optimizer → Pn / Sn ---------------------
  // thread = (4-input x 4-unit cell, row-group set): 8-row groups bgrp·NI + [0, NI)
  const int bcell = tid % (4 * U), bgrp = tid / (4 * U);
  const int dq = bcell % 16, buq = bcell / 16;
  // partial of (d = 4dq + dd, units 4buq..) at float4 slot (bgrp·CW + buq)·64 +
  // 4dq + (dd ^ ((dq >> 1) & 3)): the store of 16 lanes fills two wavefronts
  const int sw = (dq >> 1) & 3;
  // the dZ0 operand does not change across chunks: keep this thread's slice
  // in registers (NI <= 2) so a row costs one shared load per 16 FMA
  constexpr bool DZR = NI <= 2;
  float4 dzr[DZR ? NI : 1][8];
  if constexpr (DZR) {
#pragma unroll
    for (int it = 0; it < NI; ++it)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int r = 8 * (bgrp * NI + it) + j;
        dzr[it][j] = r < R ? *reinterpret_cast<const float4*>(sdZ + r * U + 4 * buq)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
      }
  }
  if (work) {
    for (int c = 0; c < nch; ++c) {
      cp_wait_n(issued_b - c - 1);
      __syncthreads();  // chunk c landed; chunk c-1's optimizer pass is done
      if (c >= 1 && c - 1 + Sb < nch) issue_b(c - 1 + Sb);
      const float* X = ring + (c % Sb) * SB;
      const float* W = X + RP * X_LD;
      const int k0 = c * X_KC, nk = min(X_KC, D - k0);
      float bacc[NI][16];
#pragma unroll
      for (int i = 0; i < NI; ++i)
#pragma unroll
        for (int e = 0; e < 16; ++e) bacc[i][e] = 0.f;
      if (4 * dq < nk) {
        const float* Xd = X + 4 * dq;
        const float* Zd = sdZ + 4 * buq;
#pragma unroll
        for (int it = 0; it < NI; ++it) {
          const int rb = 8 * (bgrp * NI + it);
          auto row = [&](int r) {
            const float4 xv = *reinterpret_cast<const float4*>(Xd + r * X_LD);
            float4 dv;
            if constexpr (DZR) dv = dzr[it][r - rb];
            else dv = *reinterpret_cast<const float4*>(Zd + r * U);
            const float xs[4] = {xv.x, xv.y, xv.z, xv.w};
            const float ds[4] = {dv.x, dv.y, dv.z, dv.w};
#pragma unroll
            for (int dd = 0; dd < 4; ++dd)
#pragma unroll
              for (int uu = 0; uu < 4; ++uu)
                bacc[it][4 * dd + uu] = fmaf(xs[dd], ds[uu], bacc[it][4 * dd + uu]);
          };
          if (rb + 8 <= R) {
#pragma unroll
            for (int j = 0; j < 8; ++j) row(rb + j);
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (rb + j < R) row(rb + j);
          }
        }
      }
      float4* red4 = reinterpret_cast<float4*>(sRed);
#pragma unroll
      for (int dd = 0; dd < 4; ++dd)
        red4[(bgrp * CW + buq) * 64 + 4 * dq + (dd ^ sw)] =
            make_float4(x_fold<NI>(bacc, 4 * dd), x_fold<NI>(bacc, 4 * dd + 1),
                        x_fold<NI>(bacc, 4 * dd + 2), x_fold<NI>(bacc, 4 * dd + 3));
      __syncthreads();
      // optimizer pass: lane pairs (j even/odd) on 16 consecutive rows d → full
      // 32-byte sectors to HBM, conflict-free shared reads
#pragma unroll
      for (int e0 = 0; e0 < 64 * CW; e0 += NT) {
        const int e = e0 + tid;
        const int jb = e & 1, d = (e >> 1) & 63, j = 2 * (e >> 7) + jb;
        if (d >= nk || 4 * j >= nu) continue;
        const int dq2 = d >> 2, dd2 = d & 3;
        float4 g = x_tree<GB>(red4 + j * 64 + 4 * dq2 + (dd2 ^ ((dq2 >> 1) & 3)), CW * 64);
        if (fault == 2) g = make_float4(NAN, NAN, NAN, NAN);
        badW0 |= !finite(g.x) | !finite(g.y) | !finite(g.z) | !finite(g.w);
        float4 w = *reinterpret_cast<const float4*>(W + d * WLD + 4 * j);
        float4 s0 = ns >= 1 ? *reinterpret_cast<const float4*>(W + X_KC * WLD + d * WLD + 4 * j)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
        float4 s1 = ns >= 2 ? *reinterpret_cast<const float4*>(W + 2 * X_KC * WLD + d * WLD + 4 * j)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
        opt_step4(OPT, lr, wd, bc1, bc2, w, s0, s1, g);
        const int64_t i = w0 + (int64_t)(k0 + d) * H + u0 + 4 * j;
        *reinterpret_cast<float4*>(Pn + i) = w;
        if (ns >= 1) *reinterpret_cast<float4*>(Sn + i) = s0;
        if (ns >= 2) *reinterpret_cast<float4*>(Sn + NP + i) = s1;
      }
    }
  }
  PK_TRACE(4);
  if (badW1) flag_min(&M.ctl->bad_grad, 0);
  if (badb1) flag_min(&M.ctl->bad_grad, 1);
  if (badW0) flag_min(&M.ctl->bad_grad, 2);
  if (badb0) flag_min(&M.ctl->bad_grad, 3);
  umma::cluster_wait();  // peers have finished reading this CTA's partials
}

// one instantiation per (rows pad, blocks per CTA): every index is a constant
__device__ void m1x_step(char* sm, const MemberDev<float>& M, const FeedDev<float>& f, int q,
                         int bpc, int Sb) {
  switch (m1_rows_pad(M.max_rows) * 8 + bpc) {
    case 32 * 8 + 1: m1x_step_t<32, 1>(sm, M, f, q, Sb); break;
    case 32 * 8 + 2: m1x_step_t<32, 2>(sm, M, f, q, Sb); break;
    case 32 * 8 + 4: m1x_step_t<32, 4>(sm, M, f, q, Sb); break;
    case 64 * 8 + 1: m1x_step_t<64, 1>(sm, M, f, q, Sb); break;
    case 64 * 8 + 2: m1x_step_t<64, 2>(sm, M, f, q, Sb); break;
    default: __trap();
  }
}
