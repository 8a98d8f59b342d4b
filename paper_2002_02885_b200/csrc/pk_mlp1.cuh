// pk_mlp1.cuh — fused packed step for one-hidden-layer members (included by
// pk_kernels.cuh).  This is the shape of every BASELINE MLP config and of the
// reference's Hyperband executor (EngineExecutor(hidden=(16,)), tuner.py:424).
//
// The hidden layer of member k is split into column blocks of BC = 8 units;
// one CTA owns block cb of one member for the whole step, so W0[:, block],
// its optimizer slots and W1[block, :] are touched by exactly one CTA:
//
//   k_mlp1_fwd   Z0/A0[:, block] = act(X·W0[:, block] + b0[block]) — X rows
//                gathered through the epoch order — and the block's partial
//                logits P_cb = A0[:, block]·W1[block, :] → global
//   k_mlp1_bwd   (launched early by PDL: prefetches W0/W1 blocks + slots and
//                the first X chunks while k_mlp1_fwd drains)
//                logits = Σ_cb P_cb + b1 (fixed cb order), softmax-xent,
//                dZ1, dZ0[:, block] = (dZ1·W1[block, :]ᵀ) ⊙ act'(Z0),
//                W1[block, :] / b1 / b0[block] updates, and the weight
//                gradient X^T·dZ0[:, block] consumed directly by the
//                optimizer against the resident W0 block.
//
// The only cross-CTA exchange is the [R x C] partial-logit block per CTA.
// Arithmetic order depends only on the member's own shape (D, H, C,
// max_rows), so packed == standalone bit for bit.

// (included inside namespace pk)

constexpr int M1_BC = 8;       // hidden units per CTA
constexpr int M1_KC = 32;      // reduction chunk over the input dimension
constexpr int M1_STAGES = 4;   // X chunks in flight
constexpr int M1_MAXR = 128;   // max rows (batch) on this path
constexpr int M1_MAXC = 32;    // max classes on this path

// rows padded to 32 / 64 / 128: fixes the thread mapping per member shape
__host__ __device__ inline int m1_rows_pad(int max_rows) {
  return max_rows <= 32 ? 32 : (max_rows <= 64 ? 64 : 128);
}

template <typename T>
struct M1 {
  static constexpr int VEC = 16 / (int)sizeof(T);
  static constexpr int XLD = M1_KC + VEC;  // padded smem row of an X chunk
  // smem bytes of each kernel for a member (D inputs, C classes, rows RP, ns slots)
  __host__ __device__ static int fwd_smem(int D, int C, int RP) {
    return M1_STAGES * (RP * XLD + M1_KC * M1_BC) * (int)sizeof(T)  // X + W0 chunk pipeline
           + (128 / RP) * RP * M1_BC * (int)sizeof(T)                // split-K partials
           + RP * M1_BC * (int)sizeof(T)                            // A0 block
           + M1_BC * C * (int)sizeof(T) + RP * 4;                   // W1 rows, row index
  }
  __host__ __device__ static int bwd_smem(int D, int C, int RP, int ns) {
    return D * M1_BC * (1 + ns) * (int)sizeof(T)      // resident W0 block + slots
           + M1_STAGES * RP * XLD * (int)sizeof(T)     // X chunk pipeline
           + RP * (M1_MAXC + 1) * (int)sizeof(T)       // logits → dlogits
           + 2 * RP * M1_BC * (int)sizeof(T)           // dZ0 block, A0 block
           + M1_BC * C * (1 + ns) * (int)sizeof(T)     // W1 rows + slots
           + 2 * RP * 4;                               // row index, labels
  }
};

template <typename T>
__device__ __forceinline__ void m1_stage_x(T* sX, const FeedDev<T>& f, const int32_t* srow,
                                           int RP, int R, int D, int k0, bool vec) {
  // X rows [0, RP) x columns [k0, k0 + KC) → sX[r][0..KC)
  constexpr int VEC = M1<T>::VEC, XLD = M1<T>::XLD;
  if (vec) {
    for (int e = threadIdx.x; e < RP * (M1_KC / VEC); e += NT) {
      const int r = e / (M1_KC / VEC), kk = (e % (M1_KC / VEC)) * VEC;
      const bool ok = r < R && k0 + kk < D;
      const T* g = ok ? f.feat + (int64_t)srow[r] * f.ld + k0 + kk : f.feat;
      cp_async<16>(sX + r * XLD + kk, g, ok);
    }
  } else {
    for (int e = threadIdx.x; e < RP * M1_KC; e += NT) {
      const int r = e / M1_KC, kk = e % M1_KC;
      const bool ok = r < R && k0 + kk < D;
      const T* g = ok ? f.feat + (int64_t)srow[r] * f.ld + k0 + kk : f.feat;
      cp_async<sizeof(T)>(sX + r * XLD + kk, g, ok);
    }
  }
}

// member-block partial logits buffer: [nb][max_rows][C] inside the Z[1] slab
// region reused as scratch (the phase path's Z_1 buffer is [max_rows][C]);
// the runtime allocates M.Z[1] with nb * max_rows * C elements for these members.

// ------------------------------------------------------------ forward --
template <typename T>
__device__ void m1_fwd_tile(char* sm, const MemberDev<T>& M, const FeedDev<T>& f, int cb) {
  const int D = M.dims[0], H = M.dims[1], C = M.dims[2];
  const int R = f.take, RP = m1_rows_pad(M.max_rows);
  const int SK = 128 / RP;               // split-K slices (fixed by RP)
  const int TPS = NT / SK;               // threads per slice = 2 * RP
  constexpr int XLD = M1<T>::XLD;
  T* sX = reinterpret_cast<T*>(sm);                         // [STAGES][RP][XLD]
  T* sB = sX + M1_STAGES * RP * XLD;                       // [STAGES][KC][BC]
  T* sRed = sB + M1_STAGES * M1_KC * M1_BC;                // [SK][RP][BC]
  T* sA0 = sRed + SK * RP * M1_BC;                          // [RP][BC]
  T* sW1 = sA0 + RP * M1_BC;                                // [BC][C]
  int32_t* srow = reinterpret_cast<int32_t*>(sW1 + M1_BC * C);
  const int par = M.ctl->parity;
  const T* P = M.params[par];
  const T* W0 = P + M.w_off[0];
  const T* b0 = P + M.b_off[0];
  const T* W1 = P + M.w_off[1];
  const int j0 = cb * M1_BC;
  for (int r = threadIdx.x; r < RP; r += NT) srow[r] = r < R ? (int32_t)feed_row(f, r) : 0;
  for (int e = threadIdx.x; e < M1_BC * C; e += NT) {
    const int j = e / C, c = e % C;
    sW1[e] = (j0 + j < H) ? W1[(int64_t)(j0 + j) * C + c] : T(0);
  }
  __syncthreads();
  PK_TRACE(1);
  const bool vx = ((reinterpret_cast<uintptr_t>(f.feat) & 15) == 0) && f.ld % M1<T>::VEC == 0 &&
                  D % M1<T>::VEC == 0;
  const bool vw = ((reinterpret_cast<uintptr_t>(W0) & 15) == 0) && H % M1<T>::VEC == 0;
  auto load = [&](int stage, int chunk) {
    const int k0 = chunk * M1_KC;
    m1_stage_x(sX + stage * RP * XLD, f, srow, RP, R, D, k0, vx);
    T* b = sB + stage * M1_KC * M1_BC;
    if (vw) {
      for (int e = threadIdx.x; e < M1_KC * (M1_BC / M1<T>::VEC); e += NT) {
        const int kk = e / (M1_BC / M1<T>::VEC), jj = (e % (M1_BC / M1<T>::VEC)) * M1<T>::VEC;
        const bool ok = k0 + kk < D && j0 + jj < H;
        cp_async<16>(b + kk * M1_BC + jj, ok ? W0 + (int64_t)(k0 + kk) * H + j0 + jj : W0, ok);
      }
    } else {
      for (int e = threadIdx.x; e < M1_KC * M1_BC; e += NT) {
        const int kk = e / M1_BC, jj = e % M1_BC;
        const bool ok = k0 + kk < D && j0 + jj < H;
        cp_async<sizeof(T)>(b + e, ok ? W0 + (int64_t)(k0 + kk) * H + j0 + jj : W0, ok);
      }
    }
  };
  // micro-tile: 2 rows x 2 cols per thread; slice s reduces k in
  // [s*KC/SK, (s+1)*KC/SK) of every chunk
  const int slice = threadIdx.x / TPS, lt = threadIdx.x % TPS;
  const int tc = lt % (M1_BC / 2), tr = lt / (M1_BC / 2);  // tr in [0, RP/2)
  const int KS = M1_KC / SK;
  T acc[2][2] = {{T(0), T(0)}, {T(0), T(0)}};
  bool badx = false;
  const int nch = (D + M1_KC - 1) / M1_KC;
  for (int s = 0; s < M1_STAGES - 1; ++s) {
    if (s < nch) load(s, s);
    cp_commit();
  }
  for (int c = 0; c < nch; ++c) {
    if (c + M1_STAGES - 1 < nch) load((c + M1_STAGES - 1) % M1_STAGES, c + M1_STAGES - 1);
    cp_commit();
    cp_wait<M1_STAGES - 1>();
    __syncthreads();
    const T* x = sX + (c % M1_STAGES) * RP * XLD;
    const T* w = sB + (c % M1_STAGES) * M1_KC * M1_BC;
#pragma unroll 4
    for (int q = 0; q < KS; ++q) {
      const int kk = slice * KS + q;
      const T a0 = x[tr * XLD + kk], a1 = x[(tr + RP / 2) * XLD + kk];
      const T w0 = w[kk * M1_BC + tc], w1 = w[kk * M1_BC + tc + M1_BC / 2];
      badx |= !finite(a0) | !finite(a1);
      acc[0][0] = fma(a0, w0, acc[0][0]);
      acc[0][1] = fma(a0, w1, acc[0][1]);
      acc[1][0] = fma(a1, w0, acc[1][0]);
      acc[1][1] = fma(a1, w1, acc[1][1]);
    }
    __syncthreads();
  }
  cp_wait<0>();
  sRed[(slice * RP + tr) * M1_BC + tc] = acc[0][0];
  sRed[(slice * RP + tr) * M1_BC + tc + M1_BC / 2] = acc[0][1];
  sRed[(slice * RP + tr + RP / 2) * M1_BC + tc] = acc[1][0];
  sRed[(slice * RP + tr + RP / 2) * M1_BC + tc + M1_BC / 2] = acc[1][1];
  badx = __syncthreads_or(badx);
  PK_TRACE(2);
  int bad = badx ? 0 : INT_MAX;
  for (int e = threadIdx.x; e < RP * M1_BC; e += NT) {
    const int r = e / M1_BC, j = e % M1_BC;
    T z = sRed[r * M1_BC + j];
    for (int s = 1; s < SK; ++s) z += sRed[(s * RP + r) * M1_BC + j];
    T a = T(0);
    if (r < R && j0 + j < H) {
      z += b0[j0 + j];
      a = act_fwd(M.act, z);
      M.Z[0][(int64_t)r * H + j0 + j] = z;
      M.A[0][(int64_t)r * H + j0 + j] = a;
      if (!finite(z)) bad = min(bad, 1);
      if (!finite(a)) bad = min(bad, 2);
    }
    sA0[r * M1_BC + j] = a;  // zero for pad rows / pad units
  }
  if (bad != INT_MAX) flag_min(&M.ctl->bad_node, bad);
  __syncthreads();
  // partial logits of this block: P[r][c] = Σ_j A0[r][j] W1[j0+j][c]
  T* part = M.Z[1] + (int64_t)cb * M.max_rows * C;
  for (int e = threadIdx.x; e < R * C; e += NT) {
    const int r = e / C, c = e % C;
    T p = T(0);
#pragma unroll
    for (int j = 0; j < M1_BC; ++j) p = fma(sA0[r * M1_BC + j], sW1[j * C + c], p);
    part[e] = p;
  }
}

// ----------------------------------------------------------- backward --
template <typename T>
__device__ void m1_bwd_tile(char* sm, const MemberDev<T>& M, const FeedDev<T>& f, int cb,
                            int nb) {
  const int D = M.dims[0], H = M.dims[1], C = M.dims[2];
  const int R = f.take, RP = m1_rows_pad(M.max_rows), ns = M.n_slots;
  constexpr int XLD = M1<T>::XLD;
  const MemberCtl* ctl = M.ctl;
  const int par = ctl->parity;
  const int64_t NP = M.s_stride;  // slot block stride
  const T* __restrict__ Pc = M.params[par];
  T* __restrict__ Pn = M.params[par ^ 1];
  const T* __restrict__ Sc = M.slots[par];
  T* __restrict__ Sn = M.slots[par ^ 1];
  const int j0 = cb * M1_BC;
  const int nj = min(M1_BC, H - j0);
  // smem carve
  T* sW0 = reinterpret_cast<T*>(sm);                     // [1+ns][D][BC]
  T* sX = sW0 + (1 + ns) * D * M1_BC;                    // [STAGES][RP][XLD]
  T* sL = sX + M1_STAGES * RP * XLD;                     // [RP][MAXC+1]
  T* sdZ0 = sL + RP * (M1_MAXC + 1);                     // [RP][BC]
  T* sA0 = sdZ0 + RP * M1_BC;                            // [RP][BC]
  T* sW1 = sA0 + RP * M1_BC;                             // [1+ns][BC][C]
  int32_t* srow = reinterpret_cast<int32_t*>(sW1 + (1 + ns) * M1_BC * C);
  int32_t* ylab = srow + RP;
  // ---- prologue: everything that does not depend on k_mlp1_fwd ----------
  for (int r = threadIdx.x; r < RP; r += NT) {
    srow[r] = r < R ? (int32_t)feed_row(f, r) : 0;
    ylab[r] = r < R ? f.labels[feed_row(f, r)] : 0;
  }
  for (int s = 0; s <= ns; ++s) {  // W0[:, block] and its slots, resident
    const T* src = (s == 0 ? Pc : Sc + (int64_t)(s - 1) * NP) + M.w_off[0];
    T* dst = sW0 + (int64_t)s * D * M1_BC;
    for (int e = threadIdx.x; e < D * M1_BC; e += NT) {
      const int k = e / M1_BC, j = e % M1_BC;
      cp_async<sizeof(T)>(dst + e, j < nj ? src + (int64_t)k * H + j0 + j : src, j < nj);
    }
    const T* s1 = (s == 0 ? Pc : Sc + (int64_t)(s - 1) * NP) + M.w_off[1];
    T* d1 = sW1 + s * M1_BC * C;
    for (int e = threadIdx.x; e < M1_BC * C; e += NT) {
      const int j = e / C;
      cp_async<sizeof(T)>(d1 + e, j < nj ? s1 + (int64_t)j0 * C + e : s1, j < nj);
    }
  }
  cp_commit();
  __syncthreads();  // srow ready for the X loads
  const bool vx = ((reinterpret_cast<uintptr_t>(f.feat) & 15) == 0) && f.ld % M1<T>::VEC == 0 &&
                  D % M1<T>::VEC == 0;
  const int nch = (D + M1_KC - 1) / M1_KC;
  for (int s = 0; s < M1_STAGES - 1; ++s) {
    if (s < nch) m1_stage_x(sX + s * RP * XLD, f, srow, RP, R, D, s * M1_KC, vx);
    cp_commit();
  }
  pdl_wait();  // k_mlp1_fwd results (partials, Z0/A0) are now visible
  PK_TRACE(1);
  // ---- logits = Σ_cb partials + b1, softmax-xent → dZ1 (in sL) -----------
  const T* part = M.Z[1];
  const T* b1 = Pc + M.b_off[1];
  int bad = INT_MAX;
  for (int e = threadIdx.x; e < R * C; e += NT) {
    const int r = e / C, c = e % C;
    T z = part[e];
    for (int q = 1; q < nb; ++q) z += part[(int64_t)q * M.max_rows * C + e];
    z += b1[c];
    sL[r * (M1_MAXC + 1) + c] = z;
    if (!finite(z)) bad = 3;
  }
  for (int e = threadIdx.x; e < RP * M1_BC; e += NT) {
    const int r = e / M1_BC, j = e % M1_BC;
    sA0[e] = (r < R && j < nj) ? M.A[0][(int64_t)r * H + j0 + j] : T(0);
  }
  if (cb == 0 && bad != INT_MAX) flag_min(&M.ctl->bad_node, bad);
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  for (int r = warp; r < R; r += NT / 32) {
    T* row = sL + r * (M1_MAXC + 1);
    xent_row(row, row, C, ylab[r], R, true, cb == 0 ? M.rowloss + r : nullptr);
  }
  __syncthreads();
  PK_TRACE(2);
  // ---- dZ0[:, block] = (dZ1 · W1[block, :]ᵀ) ⊙ act'(Z0, A0) --------------
  cp_wait<M1_STAGES - 1>();  // W0/W1 blocks (oldest group) landed
  __syncthreads();
  for (int e = threadIdx.x; e < RP * M1_BC; e += NT) {
    const int r = e / M1_BC, j = e % M1_BC;
    T v = T(0);
    if (r < R && j < nj) {
      T s = T(0);
      for (int c = 0; c < C; ++c) s = fma(sL[r * (M1_MAXC + 1) + c], sW1[j * C + c], s);
      v = act_bwd(M.act, M.Z[0][(int64_t)r * H + j0 + j], sA0[e], s);
    }
    sdZ0[e] = v;
  }
  __syncthreads();
  const T lr = T(ctl->lr), wd = T(M.wd);
  const T bc1 = M.opt == PK_OPT_ADAM ? T(ctl->bc1) : T(1);
  const T bc2 = M.opt == PK_OPT_ADAM ? T(ctl->bc2) : T(1);
  const int fault = ctl->fault_grad;
  bool badW1 = false, badb1 = false, badW0 = false, badb0 = false;
  // ---- W1[block, :] (grad position 0), b1 (1, block 0), b0[block] (3) ------
  for (int e = threadIdx.x; e < nj * C; e += NT) {
    const int j = e / C, c = e % C;
    T g = T(0);
    for (int r = 0; r < R; ++r) g = fma(sA0[r * M1_BC + j], sL[r * (M1_MAXC + 1) + c], g);
    if (fault == 0) g = T(NAN);
    badW1 |= !finite(g);
    T w = sW1[e], s0 = ns >= 1 ? sW1[M1_BC * C + e] : T(0), s1 = ns >= 2 ? sW1[2 * M1_BC * C + e] : T(0);
    opt_step(M.opt, lr, wd, bc1, bc2, w, s0, s1, g);
    const int64_t i = M.w_off[1] + (int64_t)j0 * C + e;
    Pn[i] = w;
    if (ns >= 1) Sn[i] = s0;
    if (ns >= 2) Sn[NP + i] = s1;
  }
  if (cb == 0) {
    for (int c = threadIdx.x; c < C; c += NT) {
      T g = T(0);
      for (int r = 0; r < R; ++r) g += sL[r * (M1_MAXC + 1) + c];
      if (fault == 1) g = T(NAN);
      badb1 |= !finite(g);
      const int64_t i = M.b_off[1] + c;
      T w = Pc[i], s0 = ns >= 1 ? Sc[i] : T(0), s1 = ns >= 2 ? Sc[NP + i] : T(0);
      opt_step(M.opt, lr, wd, bc1, bc2, w, s0, s1, g);
      Pn[i] = w;
      if (ns >= 1) Sn[i] = s0;
      if (ns >= 2) Sn[NP + i] = s1;
    }
  }
  for (int j = threadIdx.x; j < nj; j += NT) {
    T g = T(0);
    for (int r = 0; r < R; ++r) g += sdZ0[r * M1_BC + j];
    if (fault == 3) g = T(NAN);
    badb0 |= !finite(g);
    const int64_t i = M.b_off[0] + j0 + j;
    T w = Pc[i], s0 = ns >= 1 ? Sc[i] : T(0), s1 = ns >= 2 ? Sc[NP + i] : T(0);
    opt_step(M.opt, lr, wd, bc1, bc2, w, s0, s1, g);
    Pn[i] = w;
    if (ns >= 1) Sn[i] = s0;
    if (ns >= 2) Sn[NP + i] = s1;
  }
  PK_TRACE(3);
  // ---- W0[:, block] (grad position 2): X^T·dZ0 chunk by chunk -------------
  // thread → (k in chunk, unit pair); sum over rows in order r = 0..R-1
  for (int c = 0; c < nch; ++c) {
    if (c + M1_STAGES - 1 < nch)
      m1_stage_x(sX + ((c + M1_STAGES - 1) % M1_STAGES) * RP * XLD, f, srow, RP, R, D,
                 (c + M1_STAGES - 1) * M1_KC, vx);
    cp_commit();
    cp_wait<M1_STAGES - 1>();
    __syncthreads();
    const T* x = sX + (c % M1_STAGES) * RP * XLD;
    for (int e = threadIdx.x; e < M1_KC * M1_BC; e += NT) {
      const int kk = e / M1_BC, j = e % M1_BC;
      const int k = c * M1_KC + kk;
      if (k >= D || j >= nj) continue;
      T g = T(0);
      for (int r = 0; r < R; ++r) g = fma(x[r * XLD + kk], sdZ0[r * M1_BC + j], g);
      if (fault == 2) g = T(NAN);
      badW0 |= !finite(g);
      const int se = k * M1_BC + j;
      T w = sW0[se];
      T s0 = ns >= 1 ? sW0[D * M1_BC + se] : T(0);
      T s1 = ns >= 2 ? sW0[2 * D * M1_BC + se] : T(0);
      opt_step(M.opt, lr, wd, bc1, bc2, w, s0, s1, g);
      const int64_t i = M.w_off[0] + (int64_t)k * H + j0 + j;
      Pn[i] = w;
      if (ns >= 1) Sn[i] = s0;
      if (ns >= 2) Sn[NP + i] = s1;
    }
    __syncthreads();
  }
  cp_wait<0>();
  PK_TRACE(4);
  if (badW1) flag_min(&M.ctl->bad_grad, 0);
  if (badb1) flag_min(&M.ctl->bad_grad, 1);
  if (badW0) flag_min(&M.ctl->bad_grad, 2);
  if (badb0) flag_min(&M.ctl->bad_grad, 3);
}
