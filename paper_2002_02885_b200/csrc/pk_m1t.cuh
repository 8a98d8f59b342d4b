// pk_m1t.cuh — tensor-core (tcgen05, 3xTF32) packed step for one-hidden-layer
// fp32 members (included by pk_kernels.cuh inside namespace pk).
//
// Same math and commit rules as pk_mlp1.cuh (reference engine.py:180-326 for
// MLP [D, H, C]), but the two GEMMs that carry the step's FLOPs and its
// dominant HBM stream run on the 5th-generation tensor cores:
//
//   k_m1t_fwd  (member, 128-unit tile, 64-deep input split) per CTA:
//              TMEM[128 units x RP rows] = W0[split, tile]ᵀ · X[rows, split]ᵀ
//              W0 rows and the gathered X rows arrive by 16-byte cp.async
//              into shared memory; one staging pass splits them into
//              tf32 hi/lo K-major operands; one thread issues
//              3 x 8 tcgen05.mma.kind::tf32 (A_hi·B_hi + A_hi·B_lo + A_lo·B_hi).
//              The splits of a tile form one thread-block cluster; partials
//              stay in shared memory and are reduced over DSMEM in rank order
//              (b0, activation → Z0, A0; then the tile's partial logits per
//              member-local 32-unit block).
//   k_m1t_bwd  (member, 128-input tile, 32-unit tile) per CTA; prologue
//              (before griddepcontrol.wait, overlapping k_m1t_fwd): bulk
//              copies of W0[tile] + optimizer slots, W1 rows + slots and the
//              tile's X columns.  Then logits = Σ_blocks partials + b1,
//              softmax-xent (dZ1), dZ0 = (dZ1·W1ᵀ) ⊙ act'(Z0), and
//              TMEM[128 inputs x 32 units] = X[:, tile]ᵀ · dZ0[:, units]
//              (3xTF32, 32 rows per K chunk).  The epilogue reads the weight
//              gradient from TMEM and applies the member's optimizer against
//              the resident W0 tile — the gradient never reaches HBM.
//              Input-tile 0 CTAs also update W1 rows / b0 (and b1 in unit
//              tile 0) with the same fixed-order sums as pk_mlp1.cuh.
//
// Determinism / K-invariance: every output element is one MMA accumulation
// over a k order fixed by the member's own shape (splits of 64, chunks of 32
// rows), reduced in split order; tiles never mix members, so a member's
// packed trajectory is bit-identical to its standalone one.
//
// Accuracy: 3xTF32 error ≈ 2^-21 · Σ|a·b| per output (measured 4e-7 rel on
// B200, tools/umma_selftest.cu), inside the fp32 contract rel 1e-4.

constexpr int T_UM = 128;     // fwd: hidden units per tile (MMA M)
constexpr int T_KS = 64;      // fwd: input dims per split
constexpr int T_XLD = T_KS + 4;   // fwd: raw X row stride (floats, 16B-aligned, conflict-free)
constexpr int T_BK = 128;     // bwd: input dims per tile (MMA M)
constexpr int T_BU = 32;      // bwd: hidden units per tile (MMA N)
constexpr int T_BXLD = T_BK + 4;  // bwd: raw X row stride
constexpr int T_BWLD = T_BU + 4;  // bwd: W0-tile row stride (144 B: LDS.128 by row is conflict-free)
constexpr int T_LB = 32;      // member-local partial-logit block (units)
constexpr int T_BWD_NT = 384; // k_m1t_bwd threads: 8 epilogue + 3 producer + 1 MMA warps
constexpr int T_MAXC = 32;    // classes on this path
constexpr int T_MAXR = 128;   // rows on this path
constexpr int T_MAXCS = 16;   // max cluster size (non-portable) → D <= 1024
__host__ __device__ inline int cdiv_d(int a, int b) { return (a + b - 1) / b; }

__host__ __device__ inline int t_nsplit(int D) { return (D + T_KS - 1) / T_KS; }
__host__ __device__ inline int t_ntile(int H) { return (H + T_UM - 1) / T_UM; }
__host__ __device__ inline int t_nblk(int H) { return (H + T_LB - 1) / T_LB; }

struct M1T {
  // shared-memory bytes (fp32) for a member with rows padded to RP
  __host__ __device__ static int fwd_smem(int RP, int C) {
    return T_KS * T_UM * 4              // raw W0 rows [k][unit]
           + RP * T_XLD * 4            // raw X rows
           + 2 * T_UM * T_KS * 4       // A hi/lo
           + 2 * RP * T_KS * 4         // B hi/lo
           + T_UM * C * 4 + T_UM * 4   // W1 rows, b0 slice of the tile
           + RP * 4 + 64;              // row index, barriers
    // (the partial [RP][T_UM] reuses the A hi/lo region after the MMA)
  }
  // S = input-tile stages in flight (2 when they fit, else 1)
  __host__ __device__ static int bwd_smem(int RP, int C, int ns, int S) {
    return S * (T_BK * T_BWLD * 4 + RP * T_BXLD * 4)  // W0 tile, X columns (slots: from L2)
           + 2 * T_BK * 32 * 4         // A hi/lo (one 32-row chunk)
           + 2 * T_BU * 32 * 4         // B hi/lo
           + RP * (C + 1) * 4          // logits → dZ1 (row stride C + 1)
           + 2 * RP * T_BU * 4         // dZ0 tile, A0 tile
           + (1 + ns) * T_BU * C * 4   // W1 rows + slots
           + T_MAXC * 4                // b1
           + 2 * RP * 4 + 128;         // rows, labels, 14 barriers, TMEM slot
  }
};

// e / d and e % d for a runtime d that is a power of two on full tiles
// (8 unit quads, 32 input quads): a shift on that path, a division otherwise
__device__ __forceinline__ void divmod_p2(int e, int d, int& q, int& r) {
  if ((d & (d - 1)) == 0) {
    const int s = __ffs(d) - 1;
    q = e >> s;
    r = e & (d - 1);
  } else {
    q = e / d;
    r = e - q * d;
  }
}

// four consecutive units u..u+3 of row r with their split sums z: + b0, the
// activation, Z0/A0 (one 16-byte store each), A0 into sA4 (0 outside the box)
__device__ __forceinline__ void m1_finish4(const MemberDev<float>& M, float4 z, const float* sb0,
                                           int r, int u, int R, int nu, int u0, int H,
                                           float* sA4, int* bad) {
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
  if (r < R && u < nu) {  // H % 4 == 0: a quad is valid or not as a whole
    z.x += sb0[u];
    z.y += sb0[u + 1];
    z.z += sb0[u + 2];
    z.w += sb0[u + 3];
    a = make_float4(act_fwd(M.act, z.x), act_fwd(M.act, z.y), act_fwd(M.act, z.z),
                    act_fwd(M.act, z.w));
    *reinterpret_cast<float4*>(M.Z[0] + (int64_t)r * H + u0 + u) = z;
    *reinterpret_cast<float4*>(M.A[0] + (int64_t)r * H + u0 + u) = a;
    if (!finite(z.x) || !finite(z.y) || !finite(z.z) || !finite(z.w)) *bad = min(*bad, 1);
    if (!finite(a.x) || !finite(a.y) || !finite(a.z) || !finite(a.w)) *bad = min(*bad, 2);
  }
  *reinterpret_cast<float4*>(sA4) = a;
}

// softmax-xent of one row by an aligned group of 8 lanes (classes c ≡ lane
// mod 8, C <= 32; engine.py:211-230, :252-264): z ← dlogits in place,
// −logp[y] into *rowloss.  `live` = false lanes join the shuffles only.
__device__ __forceinline__ void xent_row8(float* z, int C, int y, int R, bool live,
                                          double* rowloss) {
  const int q = threadIdx.x & 7;
  float v[4];
  float mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int c = q + 8 * i;
    v[i] = live && c < C ? z[c] : -INFINITY;  // idle lanes never touch smem
    mx = fmaxf(mx, v[i]);
  }
#pragma unroll
  for (int o = 4; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o, 8));
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (q + 8 * i < C) s = __fadd_rn(s, ex(__fsub_rn(v[i], mx)));
#pragma unroll
  for (int o = 4; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, 8);
  if (!live) return;
  const float zy = z[y];
  __syncwarp(0xffu << (threadIdx.x & 24));  // the row's 8 lanes read z[y] first
  const float inv = 1.f / s, nv = float(R);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int c = q + 8 * i;
    if (c < C) {
      float p = __fmul_rn(ex(__fsub_rn(v[i], mx)), inv);
      if (c == y) p = __fsub_rn(p, 1.f);
      z[c] = __fdiv_rn(p, nv);
    }
  }
  if (q == 0 && rowloss) *rowloss = -(double)((zy - mx) - lg(s));
}

// ------------------------------------------------------------ forward --
// One thread-block cluster per (member, 128-unit tile); cluster rank = input
// split.  Each CTA leaves its TMEM partial in its own shared memory; after a
// cluster barrier, rank q reduces member-local 32-unit block(s) q, q+CS, ...
// by reading the CS partials over DSMEM in rank order (fixed order ⇒
// deterministic), adds b0, applies the activation and writes Z0/A0 and the
// block's partial logits.
__device__ void m1t_fwd_tile(char* sm, const MemberDev<float>& M, const FeedDev<float>& f,
                             int tile, int split, int CS, const PhaseArgs<float>& P) {
  const int D = M.dims[0], H = M.dims[1], C = M.dims[2];
  const int R = f.take, RP = m1_rows_pad(M.max_rows);
  const int u0 = tile * T_UM, nu = min(T_UM, H - u0);
  const int ks = split * T_KS, nk = max(0, min(T_KS, D - ks));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  float* rawA = reinterpret_cast<float*>(sm);     // [T_KS][T_UM]
  float* rawX = rawA + T_KS * T_UM;               // [RP][T_XLD]
  float* Ah = rawX + RP * T_XLD;                  // K-major [T_KS/4][T_UM][4]
  float* Al = Ah + T_UM * T_KS;
  float* Bh = Al + T_UM * T_KS;                   // K-major [T_KS/4][RP][4]
  float* Bl = Bh + RP * T_KS;
  float* sW1 = Bl + RP * T_KS;                    // [T_UM][C] W1 rows of the tile
  float* sb0 = sW1 + T_UM * C;                    // [T_UM] b0 slice
  int32_t* srow = reinterpret_cast<int32_t*>(sb0 + T_UM);
  uint64_t* bar = reinterpret_cast<uint64_t*>(srow + RP);  // [2] (RP even)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
  float* sP = Ah;                                 // after the MMA: partial [RP][T_UM]
  const uint32_t tcols = umma::tmem_cols_pow2(RP);
  const int nu4 = (nu + 3) & ~3;
  const bool reducer = true;  // every rank reduces a row subset of the tile

  // ---- everything that does not depend on the previous step: the batch's
  //      gather index, barriers, TMEM and the X rows (inside a multi-step
  //      graph this overlaps the previous step's tail)
  const int myrow = tid < R ? (int32_t)feed_row(f, tid) : 0;
  if (tid < RP) srow[tid] = myrow;  // RP <= 128 < NT
  if (tid == 32) {
    umma::mbar_init(&bar[1], 1);
    umma::mbar_fence_init();
  }
  if (warp == 1) umma::tmem_alloc(tslot, tcols);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  {
    const int cpr = nk / 4;
    for (int e = tid; e < R * cpr; e += NT) {
      int r, c;
      divmod_p2(e, cpr, r, c);
      cp_async<16>(rawX + r * T_XLD + 4 * c, f.feat + (int64_t)srow[r] * f.ld + ks + 4 * c, true);
    }
  }
  const uint32_t tmem = *tslot;
  // ---- the member's state: after the previous step (parity, halt flag)
  if (P.first) {
    pdl_wait();
    pdl_launch();
  }
  if (halted(P)) {  // uniform over the grid: no cluster barrier is left waiting
    cp_wait<0>();
    umma::fence_before();
    __syncthreads();
    if (warp == 1) umma::tmem_dealloc(tmem, tcols);
    return;
  }
  const float* Pc = M.params[M.ctl->parity];
  const float* W0 = Pc + M.w_off[0];
  {
    const int cpr = nu4 / 4;
    for (int e = tid; e < nk * cpr; e += NT) {
      int k, c;
      divmod_p2(e, cpr, k, c);
      cp_async<16>(rawA + k * T_UM + 4 * c, W0 + (int64_t)(ks + k) * H + u0 + 4 * c, true);
    }
    if (reducer) {
      for (int e = tid; e < nu4 * C / 4; e += NT)
        cp_async<16>(sW1 + 4 * e, Pc + M.w_off[1] + (int64_t)u0 * C + 4 * e, true);
      for (int e = tid; e < cpr; e += NT) cp_async<16>(sb0 + 4 * e, Pc + M.b_off[0] + u0 + 4 * e, true);
    }
  }
  cp_commit();
  PK_TRACE(1);
  cp_wait<0>();
  __syncthreads();
  if (nk > 0) {
    // split pass → tf32 hi/lo K-major operands (zero outside the valid box)
    for (int e = tid; e < T_UM * (T_KS / 4); e += NT) {
      const int u = e % T_UM, kq = e / T_UM;
      float4 h, l;
      float* hp = &h.x;
      float* lp = &l.x;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int k = 4 * kq + j;
        const float v = (u < nu && k < nk) ? rawA[k * T_UM + u] : 0.f;
        umma::split3(v, hp[j], lp[j]);
      }
      const uint32_t o = umma::kmaj_off(u, 4 * kq, T_UM) / 4;
      *reinterpret_cast<float4*>(Ah + o) = h;
      *reinterpret_cast<float4*>(Al + o) = l;
    }
    bool badx = false;
    for (int e = tid; e < RP * (T_KS / 4); e += NT) {
      const int r = e % RP, kq = e / RP;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < R && 4 * kq < nk) v = *reinterpret_cast<const float4*>(rawX + r * T_XLD + 4 * kq);
      badx |= !finite(v.x) | !finite(v.y) | !finite(v.z) | !finite(v.w);
      float4 h, l;
      umma::split3(v.x, h.x, l.x);
      umma::split3(v.y, h.y, l.y);
      umma::split3(v.z, h.z, l.z);
      umma::split3(v.w, h.w, l.w);
      const uint32_t o = umma::kmaj_off(r, 4 * kq, RP) / 4;
      *reinterpret_cast<float4*>(Bh + o) = h;
      *reinterpret_cast<float4*>(Bl + o) = l;
    }
    umma::fence_async_smem();
    umma::fence_before();
    badx = __syncthreads_or(badx);
    umma::fence_after();
    if (badx && tid == 0) flag_min(&M.ctl->bad_node, 0);
    if (tid == 0) {
      const uint32_t idesc = umma::idesc_tf32(T_UM, RP, false, false);
      const uint32_t ah = umma::smem_u32(Ah), al = umma::smem_u32(Al);
      const uint32_t bh = umma::smem_u32(Bh), bl = umma::smem_u32(Bl);
      const int nks = (nk + 7) / 8;
      for (int s = 0; s < nks; ++s) {
        const uint64_t dah = umma::kmaj_desc(ah, T_UM, s), dal = umma::kmaj_desc(al, T_UM, s);
        const uint64_t dbh = umma::kmaj_desc(bh, RP, s), dbl = umma::kmaj_desc(bl, RP, s);
        umma::mma_tf32(tmem, dah, dbh, idesc, s > 0);
        umma::mma_tf32(tmem, dah, dbl, idesc, true);
        umma::mma_tf32(tmem, dal, dbh, idesc, true);
      }
      umma::commit(&bar[1]);
    }
    umma::mbar_wait(&bar[1], 0);
    umma::fence_after();
  }
  PK_TRACE(2);
  __syncthreads();  // every thread is past the MMA: Ah/Al may be overwritten
  // TMEM partial → own shared memory sP[r][u] (rows r < R; zeros if no split)
  {
    const int q = warp & 3, half = warp >> 2;
    const int u = 32 * q + lane;
    for (int c = half * (RP / 2); c < (half + 1) * (RP / 2); c += 8) {
      float v[8];
      if (nk > 0) {
        umma::tmem_ld8(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)c, v);
        umma::tmem_wait_ld();
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = 0.f;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) sP[(c + i) * T_UM + u] = v[i];
    }
  }
  umma::fence_before();
  umma::cluster_sync();  // all partials of the tile are in the cluster's shared memory
  PK_TRACE(3);
  if (warp == 1) umma::tmem_dealloc(tmem, tcols);
  // ---- rank q reduces rows q, q + CS, ... (all units of the tile): every CTA
  //      of the cluster shares the epilogue ----------------------------------
  float* sA = rawA;  // [my rows][T_UM] activations (rawA + rawX are free now)
  const int nr = R > split ? (R - split + CS - 1) / CS : 0;
  int bad = INT_MAX;
  // four consecutive units per thread: one 16-byte DSMEM load per rank
  for (int e4 = tid; e4 < nr * T_UM / 4; e4 += NT) {
    const int rl = e4 / (T_UM / 4), u = 4 * (e4 % (T_UM / 4)), r = split + rl * CS;
    float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    if (u < nu) {
      float4 v[T_MAXCS];
      const uint32_t la = umma::smem_u32(sP + r * T_UM + u);
#pragma unroll
      for (int s = 0; s < T_MAXCS; ++s)
        v[s] = s < CS ? umma::dsmem_ld4(la, (uint32_t)s) : make_float4(0.f, 0.f, 0.f, 0.f);
      z = v[0];
#pragma unroll
      for (int s = 1; s < T_MAXCS; ++s)
        if (s < CS) {
          z.x += v[s].x;
          z.y += v[s].y;
          z.z += v[s].z;
          z.w += v[s].w;
        }
    }
    m1_finish4(M, z, sb0, r, u, R, nu, u0, H, sA + rl * T_UM + u, &bad);
  }
  __syncthreads();
  // P[blk][r][c] = Σ_{j<32} A0[r][32·blk + j] · W1[32·blk + j][c] for my rows
  const int nbt = (nu + T_LB - 1) / T_LB;
  for (int e = tid; e < nbt * nr * C; e += NT) {
    const int bl = e / (nr * C), rc = e % (nr * C), rl = rc / C, c = rc % C;
    const int ub = bl * T_LB, r = split + rl * CS;
    const float* a = sA + rl * T_UM + ub;
    const float* w = sW1 + ub * C + c;  // rows u >= nu: a = 0 there
    float p = 0.f;
#pragma unroll 8
    for (int j = 0; j < T_LB; ++j) p = fmaf(a[j], ub + j < nu ? w[j * C] : 0.f, p);
    M.Z[1][((int64_t)(u0 / T_LB + bl) * M.max_rows + r) * C + c] = p;
  }
  if (bad != INT_MAX) flag_min(&M.ctl->bad_node, bad);
  PK_TRACE(4);
  umma::cluster_arrive_relaxed();  // peers are done reading this CTA's partial:
  umma::cluster_wait();            // no memory ordering needed, just the rendezvous
}

// ------------------------------------------------ streaming forward --
// For packs whose split-K clusters would need several waves: one CTA per
// (member, 128-unit tile) walks the whole input dimension.  Raw 32-deep
// chunks of W0 rows and X rows stream through an S-stage cp.async ring and
// are split into tf32 hi/lo (double-buffered) while the tensor core works on
// the previous chunk.  The arithmetic is the cluster forward's exactly: input
// split s (64 deep = chunks 2s, 2s+1) accumulates alone in TMEM buffer s & 1
// with the same MMA sequence, and its partial is read out and added into
// running registers in split order (z = p0 + p1 + ... + b0) while split s+1
// multiplies — so a member's result does not depend on which forward variant
// its pack size selected (packed == standalone stays bit-exact).
constexpr int T_SC = 32;              // input dims per streamed chunk
constexpr int T_SXLD = T_SC + 4;      // raw X chunk row stride (16B rows, conflict-free)

// sA[r][u] holds z = Σ partials + b0 for the tile's rows × units: activation,
// Z0 / A0 to global (coalesced along u), sA ← A0 (0 outside the valid box)
__device__ __forceinline__ void m1_act_epilogue(const MemberDev<float>& M, float* sA, int R, int RP,
                                                int nu, int u0, int H, int* bad) {
#pragma unroll 1
  for (int e = threadIdx.x; e < RP * T_UM; e += blockDim.x) {
    const int r = e / T_UM, u = e % T_UM;
    float a = 0.f;
    if (r < R && u < nu) {
      const float zz = sA[e];
      a = act_fwd(M.act, zz);
      M.Z[0][(int64_t)r * H + u0 + u] = zz;
      M.A[0][(int64_t)r * H + u0 + u] = a;
      if (!finite(zz)) *bad = min(*bad, 1);
      if (!finite(a)) *bad = min(*bad, 2);
    }
    sA[e] = a;
  }
}

__host__ __device__ inline int m1s_raw_stages(int RP) { return RP >= 128 ? 2 : 4; }
__host__ __device__ inline int m1s_fwd_smem(int RP, int C) {
  const int S = m1s_raw_stages(RP);
  return S * (T_SC * T_UM + RP * T_SXLD) * 4   // raw W0 / X chunks
         + 2 * 2 * (T_UM + RP) * T_SC * 4      // hi/lo A and B, double-buffered
         + T_UM * C * 4 + T_UM * 4             // W1 rows, b0 slice
         + RP * 4 + 64;                        // row index, barriers
}

__device__ void m1s_fwd_tile(char* sm, const MemberDev<float>& M, const FeedDev<float>& f,
                             int tile) {
  const int D = M.dims[0], H = M.dims[1], C = M.dims[2];
  const int R = f.take, RP = m1_rows_pad(M.max_rows), S = m1s_raw_stages(RP);
  const int u0 = tile * T_UM, nu = min(T_UM, H - u0), nu4 = (nu + 3) & ~3;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int RSF = T_SC * T_UM + RP * T_SXLD;        // floats per raw stage
  float* raw = reinterpret_cast<float*>(sm);        // [S][rawA chunk, rawX chunk]
  float* hl = raw + S * RSF;                        // [2][Ah, Al, Bh, Bl]
  const int HLF = 2 * (T_UM + RP) * T_SC;            // floats per hi/lo buffer
  float* sW1 = hl + 2 * HLF;
  float* sb0 = sW1 + T_UM * C;
  int32_t* srow = reinterpret_cast<int32_t*>(sb0 + T_UM);
  uint64_t* bar = reinterpret_cast<uint64_t*>(srow + RP);  // [0,1] hi/lo free, [2,3] split done
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 4);
  const float* Pc = M.params[M.ctl->parity];
  const float* W0 = Pc + M.w_off[0];
  const uint32_t tcols = umma::tmem_cols_pow2(2 * RP);
  const int nch = (D + T_SC - 1) / T_SC, nsplit = t_nsplit(D);

  for (int r = tid; r < RP; r += NT) srow[r] = r < R ? (int32_t)feed_row(f, r) : 0;
  if (tid == 32) {
    for (int i = 0; i < 4; ++i) umma::mbar_init(&bar[i], 1);
    umma::mbar_fence_init();
  }
  if (warp == 1) umma::tmem_alloc(tslot, tcols);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = *tslot;
  auto issue = [&](int c) {  // raw chunk c into stage c % S (one commit group)
    float* rA = raw + (c % S) * RSF;
    float* rX = rA + T_SC * T_UM;
    const int k0 = c * T_SC, nk = min(T_SC, D - k0), cpr = nu4 / 4;
    for (int e = tid; e < nk * cpr; e += NT) {
      int k, q;
      divmod_p2(e, cpr, k, q);
      cp_async<16>(rA + k * T_UM + 4 * q, W0 + (int64_t)(k0 + k) * H + u0 + 4 * q, true);
    }
    const int cx = nk / 4;
    for (int e = tid; e < R * cx; e += NT) {
      int r, q;
      divmod_p2(e, cx, r, q);
      cp_async<16>(rX + r * T_SXLD + 4 * q, f.feat + (int64_t)srow[r] * f.ld + k0 + 4 * q, true);
    }
    cp_commit();
  };
  // W1 / b0 of the tile ride in the first commit group
  for (int e = tid; e < nu4 * C / 4; e += NT)
    cp_async<16>(sW1 + 4 * e, Pc + M.w_off[1] + (int64_t)u0 * C + 4 * e, true);
  for (int e = tid; e < nu4 / 4; e += NT) cp_async<16>(sb0 + 4 * e, Pc + M.b_off[0] + u0 + 4 * e, true);
  for (int c = 0; c < S - 1; ++c) {
    if (c < nch) issue(c);
    else cp_commit();
  }
  PK_TRACE(1);
  const uint32_t idesc = umma::idesc_tf32(T_UM, RP, false, false);
  // running split sums: warp w owns TMEM lane quarter w % 4 (units) and row
  // half w / 4; RP/2 <= 64 rows per thread
  const int q = warp & 3, half = warp >> 2, uu = 32 * q + lane;
  const int rlo = half * (RP / 2);
  float z[64];
  bool badx = false;
  uint32_t ph[4] = {0u, 0u, 0u, 0u};
  auto readout = [&](int sp) {  // add split sp's partial (buffer sp & 1) into z
    const int ab = sp & 1;
    umma::mbar_wait(&bar[2 + ab], ph[2 + ab]);
    ph[2 + ab] ^= 1u;
    umma::fence_after();
#pragma unroll
    for (int c0 = 0; c0 < 64; c0 += 8) {
      if (c0 >= RP / 2) break;
      float v[8];
      umma::tmem_ld8(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(ab * RP + rlo + c0), v);
      umma::tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 8; ++i) z[c0 + i] = sp == 0 ? v[i] : z[c0 + i] + v[i];
    }
    umma::fence_before();
  };
  for (int c = 0; c < nch; ++c) {
    if (c + S - 1 < nch) issue(c + S - 1);
    else cp_commit();
    // chunk c landed: the S - 1 newer groups (chunks c+1 .. c+S-1) may fly
    if (S == 4) cp_wait<3>(); else cp_wait<1>();
    __syncthreads();
    if (c == 2) PK_TRACE(8);
    const int b = c & 1, sp = c >> 1;
    float* Ah = hl + b * HLF;
    float* Al = Ah + T_UM * T_SC;
    float* Bh = Al + T_UM * T_SC;
    float* Bl = Bh + RP * T_SC;
    if (c >= 2) {  // hi/lo buffer b was read by the MMAs of chunk c - 2
      umma::mbar_wait(&bar[b], ph[b]);
      ph[b] ^= 1u;
      umma::fence_after();
    }
    if (c == 2) PK_TRACE(9);
    const float* rA = raw + (c % S) * RSF;
    const float* rX = rA + T_SC * T_UM;
    const int nk = min(T_SC, D - c * T_SC);
    for (int e = tid; e < T_UM * (T_SC / 4); e += NT) {
      const int u = e % T_UM, kq = e / T_UM;
      float4 h, l;
      float* hp = &h.x;
      float* lp = &l.x;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int k = 4 * kq + j;
        const float v = (u < nu && k < nk) ? rA[k * T_UM + u] : 0.f;
        umma::split3(v, hp[j], lp[j]);
      }
      const uint32_t o = umma::kmaj_off(u, 4 * kq, T_UM) / 4;
      *reinterpret_cast<float4*>(Ah + o) = h;
      *reinterpret_cast<float4*>(Al + o) = l;
    }
    for (int e = tid; e < RP * (T_SC / 4); e += NT) {
      const int r = e % RP, kq = e / RP;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < R && 4 * kq < nk) v = *reinterpret_cast<const float4*>(rX + r * T_SXLD + 4 * kq);
      badx |= !finite(v.x) | !finite(v.y) | !finite(v.z) | !finite(v.w);
      float4 h, l;
      umma::split3(v.x, h.x, l.x);
      umma::split3(v.y, h.y, l.y);
      umma::split3(v.z, h.z, l.z);
      umma::split3(v.w, h.w, l.w);
      const uint32_t o = umma::kmaj_off(r, 4 * kq, RP) / 4;
      *reinterpret_cast<float4*>(Bh + o) = h;
      *reinterpret_cast<float4*>(Bl + o) = l;
    }
    if (c == 2) PK_TRACE(10);
    umma::fence_async_smem();
    umma::fence_before();
    __syncthreads();  // also: raw stage c % S is free for chunk c + S
    umma::fence_after();
    if (c == 2) PK_TRACE(11);
    // split sp - 2 used this accumulator buffer: its readout finished before
    // the __syncthreads above (readout of split sp - 1 happens below)
    if (tid == 0) {
      const uint32_t ah = umma::smem_u32(Ah), al = umma::smem_u32(Al);
      const uint32_t bh = umma::smem_u32(Bh), bl = umma::smem_u32(Bl);
      const uint32_t acc = tmem + (uint32_t)((sp & 1) * RP);
      for (int s2 = 0; s2 < (nk + 7) / 8; ++s2) {
        const uint64_t dah = umma::kmaj_desc(ah, T_UM, s2), dal = umma::kmaj_desc(al, T_UM, s2);
        const uint64_t dbh = umma::kmaj_desc(bh, RP, s2), dbl = umma::kmaj_desc(bl, RP, s2);
        umma::mma_tf32(acc, dah, dbh, idesc, (c & 1) || s2 > 0);
        umma::mma_tf32(acc, dah, dbl, idesc, true);
        umma::mma_tf32(acc, dal, dbh, idesc, true);
      }
      umma::commit(&bar[b]);                                  // hi/lo buffer b free
      if ((c & 1) || c == nch - 1) umma::commit(&bar[2 + (sp & 1)]);  // split sp done
    }
    // read out the previous split while this one multiplies
    if (c == 2) PK_TRACE(12);
    if ((c & 1) && sp >= 1) readout(sp - 1);
    if (c == 3) PK_TRACE(13);
  }
  cp_wait<0>();
  if (nsplit >= 2 && (nch & 1)) readout(nsplit - 2);  // odd tail: split nsplit-2 not read yet
  readout(nsplit - 1);
  badx = __syncthreads_or(badx);
  if (badx && tid == 0) flag_min(&M.ctl->bad_node, 0);
  PK_TRACE(2);
  // ---- epilogue: b0, activation, Z0/A0; sA[r][u] for the logits
  float* sA = raw;  // [RP][T_UM] (raw stages are free)
  // z + b0 through shared memory: the unrolled part is plain stores, the
  // activation and the Z0/A0 stores one rolled loop (compact code: this runs
  // once per step, every line of it an instruction-cache miss otherwise)
#pragma unroll
  for (int i = 0; i < 64; ++i) {
    if (i >= RP / 2) break;
    sA[(rlo + i) * T_UM + uu] = z[i] + sb0[uu];
  }
  __syncthreads();
  int bad = INT_MAX;
  m1_act_epilogue(M, sA, R, RP, nu, u0, H, &bad);
  if (bad != INT_MAX) flag_min(&M.ctl->bad_node, bad);
  umma::fence_before();
  __syncthreads();
  PK_TRACE(3);
  if (warp == 1) umma::tmem_dealloc(tmem, tcols);
  // P[blk][r][c] = Σ_{j<32} A0[r][32·blk + j] · W1[32·blk + j][c]
  const int nbt = (nu + T_LB - 1) / T_LB;
  for (int e = tid; e < nbt * R * C; e += NT) {
    const int bl = e / (R * C), rc = e % (R * C), r = rc / C, c = rc % C;
    const int ub = bl * T_LB;
    const float* a = sA + r * T_UM + ub;
    const float* w = sW1 + ub * C + c;
    float p = 0.f;
#pragma unroll 8
    for (int j = 0; j < T_LB; ++j) p = fmaf(a[j], ub + j < nu ? w[j * C] : 0.f, p);
    M.Z[1][((int64_t)(u0 / T_LB + bl) * M.max_rows + r) * C + c] = p;
  }
  PK_TRACE(4);
}

// --------------------------------- warp-specialised streaming forward --
// RP = 32 and ≤ 16 input splits: every split owns its TMEM accumulator
// (≤ 512 columns), so nothing is read out mid-loop and the roles separate:
//   warps 0-6 (producers): cp.async ring → wait → tf32 hi/lo split into
//                          buffer c & 1 → mbarrier full[c & 1]
//   warp 7, lane 0 (MMA):  wait full → 3 × K-steps tcgen05.mma into the
//                          split's accumulator → commit empty[c & 1]
// so staging chunk c+1 overlaps the MMAs of chunk c.  Same per-split MMA
// sequence and split-order sum as the cluster forward (bit-identical).
constexpr int T_WS_PRODUCERS = NT - 32;   // 224 threads

__device__ void m1s_fwd_tile_ws(char* sm, const MemberDev<float>& M, const FeedDev<float>& f,
                                int tile) {
  const int D = M.dims[0], H = M.dims[1], C = M.dims[2];
  const int R = f.take, RP = 32, S = 4;
  const int u0 = tile * T_UM, nu = min(T_UM, H - u0), nu4 = (nu + 3) & ~3;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int RSF = T_SC * T_UM + RP * T_SXLD;
  float* raw = reinterpret_cast<float*>(sm);
  float* hl = raw + S * RSF;
  const int HLF = 2 * (T_UM + RP) * T_SC;
  float* sW1 = hl + 2 * HLF;
  float* sb0 = sW1 + T_UM * C;
  int32_t* srow = reinterpret_cast<int32_t*>(sb0 + T_UM);
  uint64_t* bar = reinterpret_cast<uint64_t*>(srow + RP);  // [0,1] full, [2,3] empty, [4] done
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 5);
  const float* Pc = M.params[M.ctl->parity];
  const float* W0 = Pc + M.w_off[0];
  const int nch = (D + T_SC - 1) / T_SC, nsplit = t_nsplit(D);
  constexpr uint32_t tcols = 512;

  for (int r = tid; r < RP; r += NT) srow[r] = r < R ? (int32_t)feed_row(f, r) : 0;
  if (tid == 32) {
    umma::mbar_init(&bar[0], 7);  // one arrive per producer warp
    umma::mbar_init(&bar[1], 7);
    umma::mbar_init(&bar[2], 1);
    umma::mbar_init(&bar[3], 1);
    umma::mbar_init(&bar[4], 1);
    umma::mbar_fence_init();
  }
  if (warp == 1) umma::tmem_alloc(tslot, tcols);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = *tslot;
  bool badx = false;
  if (warp < 7) {
    // ------------------------------------------------------------ producers
    const int pt = tid;  // 0 .. 223
    auto issue = [&](int c) {
      float* rA = raw + (c % S) * RSF;
      float* rX = rA + T_SC * T_UM;
      const int k0 = c * T_SC, nk = min(T_SC, D - k0), cpr = nu4 / 4;
      for (int e = pt; e < nk * cpr; e += T_WS_PRODUCERS) {
        int k, q;
      divmod_p2(e, cpr, k, q);
        cp_async<16>(rA + k * T_UM + 4 * q, W0 + (int64_t)(k0 + k) * H + u0 + 4 * q, true);
      }
      const int cx = nk / 4;
      for (int e = pt; e < R * cx; e += T_WS_PRODUCERS) {
        int r, q;
      divmod_p2(e, cx, r, q);
        cp_async<16>(rX + r * T_SXLD + 4 * q, f.feat + (int64_t)srow[r] * f.ld + k0 + 4 * q, true);
      }
      cp_commit();
    };
    for (int e = pt; e < nu4 * C / 4; e += T_WS_PRODUCERS)
      cp_async<16>(sW1 + 4 * e, Pc + M.w_off[1] + (int64_t)u0 * C + 4 * e, true);
    for (int e = pt; e < nu4 / 4; e += T_WS_PRODUCERS)
      cp_async<16>(sb0 + 4 * e, Pc + M.b_off[0] + u0 + 4 * e, true);
    for (int c = 0; c < S - 1; ++c) {
      if (c < nch) issue(c);
      else cp_commit();
    }
    uint32_t eph[2] = {0u, 0u};
    for (int c = 0; c < nch; ++c) {
      if (c + S - 1 < nch) issue(c + S - 1);
      else cp_commit();
      cp_wait<3>();
      asm volatile("bar.sync 1, %0;" ::"n"(T_WS_PRODUCERS) : "memory");  // chunk c landed
      if (c == 8) PK_TRACE(8);
      const int b = c & 1;
      if (c >= 2) {  // buffer b consumed by the MMAs of chunk c - 2
        umma::mbar_wait(&bar[2 + b], eph[b]);
        eph[b] ^= 1u;
      }
      if (c == 8) PK_TRACE(9);
      float* Ah = hl + b * HLF;
      float* Al = Ah + T_UM * T_SC;
      float* Bh = Al + T_UM * T_SC;
      float* Bl = Bh + RP * T_SC;
      const float* rA = raw + (c % S) * RSF;
      const float* rX = rA + T_SC * T_UM;
      const int nk = min(T_SC, D - c * T_SC);
      for (int e = pt; e < T_UM * (T_SC / 4); e += T_WS_PRODUCERS) {
        const int u = e % T_UM, kq = e / T_UM;
        float4 h, l;
        float* hp = &h.x;
        float* lp = &l.x;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int k = 4 * kq + j;
          const float v = (u < nu && k < nk) ? rA[k * T_UM + u] : 0.f;
          umma::split3(v, hp[j], lp[j]);
        }
        const uint32_t o = umma::kmaj_off(u, 4 * kq, T_UM) / 4;
        *reinterpret_cast<float4*>(Ah + o) = h;
        *reinterpret_cast<float4*>(Al + o) = l;
      }
      for (int e = pt; e < RP * (T_SC / 4); e += T_WS_PRODUCERS) {
        const int r = e % RP, kq = e / RP;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (r < R && 4 * kq < nk) v = *reinterpret_cast<const float4*>(rX + r * T_SXLD + 4 * kq);
        badx |= !finite(v.x) | !finite(v.y) | !finite(v.z) | !finite(v.w);
        float4 h, l;
        umma::split3(v.x, h.x, l.x);
        umma::split3(v.y, h.y, l.y);
        umma::split3(v.z, h.z, l.z);
        umma::split3(v.w, h.w, l.w);
        const uint32_t o = umma::kmaj_off(r, 4 * kq, RP) / 4;
        *reinterpret_cast<float4*>(Bh + o) = h;
        *reinterpret_cast<float4*>(Bl + o) = l;
      }
      if (c == 8) PK_TRACE(10);
      umma::fence_async_smem();
      // every producer is past its raw-stage reads and hi/lo writes before the
      // stage is refilled (next iteration's issue) and before the MMA starts
      asm volatile("bar.sync 1, %0;" ::"n"(T_WS_PRODUCERS) : "memory");
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(umma::smem_u32(&bar[b])) : "memory");
      if (c == 8) PK_TRACE(11);
    }
    cp_wait<0>();
  } else if (lane == 0) {
    // --------------------------------------------------------- MMA issuer
    const uint32_t idesc = umma::idesc_tf32(T_UM, RP, false, false);
    uint32_t fph[2] = {0u, 0u};
    for (int c = 0; c < nch; ++c) {
      const int b = c & 1;
      umma::mbar_wait(&bar[b], fph[b]);
      fph[b] ^= 1u;
      umma::fence_after();
      if (c == 8 && pk_trace_slots) pk_trace_slots[12] = gtimer();
      float* Ah = hl + b * HLF;
      float* Al = Ah + T_UM * T_SC;
      float* Bh = Al + T_UM * T_SC;
      float* Bl = Bh + RP * T_SC;
      const uint32_t ah = umma::smem_u32(Ah), al = umma::smem_u32(Al);
      const uint32_t bh = umma::smem_u32(Bh), bl = umma::smem_u32(Bl);
      const uint32_t acc = tmem + (uint32_t)((c >> 1) * RP);
      const int nk = min(T_SC, D - c * T_SC);
      for (int s2 = 0; s2 < (nk + 7) / 8; ++s2) {
        const uint64_t dah = umma::kmaj_desc(ah, T_UM, s2), dal = umma::kmaj_desc(al, T_UM, s2);
        const uint64_t dbh = umma::kmaj_desc(bh, RP, s2), dbl = umma::kmaj_desc(bl, RP, s2);
        umma::mma_tf32(acc, dah, dbh, idesc, (c & 1) || s2 > 0);
        umma::mma_tf32(acc, dah, dbl, idesc, true);
        umma::mma_tf32(acc, dal, dbh, idesc, true);
      }
      umma::commit(&bar[2 + b]);
      if (c == 8 && pk_trace_slots) pk_trace_slots[13] = gtimer();
    }
    umma::commit(&bar[4]);
  }
  // ---- all warps: accumulators done → split-order sum, epilogue -----------
  umma::mbar_wait(&bar[4], 0);
  umma::fence_after();
  badx = __syncthreads_or(badx);
  if (badx && tid == 0) flag_min(&M.ctl->bad_node, 0);
  PK_TRACE(2);
  const int q = warp & 3, half = warp >> 2, uu = 32 * q + lane, rlo = half * (RP / 2);
  float z[16];
  for (int sp = 0; sp < nsplit; ++sp) {
#pragma unroll
    for (int c0 = 0; c0 < 16; c0 += 8) {
      float v[8];
      umma::tmem_ld8(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(sp * RP + rlo + c0), v);
      umma::tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 8; ++i) z[c0 + i] = sp == 0 ? v[i] : z[c0 + i] + v[i];
    }
  }
  float* sA = raw;  // [RP][T_UM]
#pragma unroll
  for (int i = 0; i < 16; ++i) sA[(rlo + i) * T_UM + uu] = z[i] + sb0[uu];
  __syncthreads();
  int bad = INT_MAX;
  m1_act_epilogue(M, sA, R, RP, nu, u0, H, &bad);
  if (bad != INT_MAX) flag_min(&M.ctl->bad_node, bad);
  umma::fence_before();
  __syncthreads();
  PK_TRACE(3);
  if (warp == 1) umma::tmem_dealloc(tmem, tcols);
  const int nbt = (nu + T_LB - 1) / T_LB;
  for (int e = tid; e < nbt * R * C; e += NT) {
    const int bl = e / (R * C), rc = e % (R * C), r = rc / C, c = rc % C;
    const int ub = bl * T_LB;
    const float* a = sA + r * T_UM + ub;
    const float* w = sW1 + ub * C + c;
    float p = 0.f;
#pragma unroll 8
    for (int j = 0; j < T_LB; ++j) p = fmaf(a[j], ub + j < nu ? w[j * C] : 0.f, p);
    M.Z[1][((int64_t)(u0 / T_LB + bl) * M.max_rows + r) * C + c] = p;
  }
  PK_TRACE(4);
}

// ------------------------- cluster-streaming forward (the general form) --
// One thread-block cluster of CS CTAs per (member, 128-unit tile); rank r
// owns a contiguous range of the 64-deep input splits and streams their
// 32-deep chunks through a warp-specialised pipeline (7 producer warps:
// cp.async ring → tf32 hi/lo split; 1 MMA warp).  Every split accumulates
// alone in its own TMEM columns with the cluster forward's MMA sequence; the
// partials land in the CTA's shared memory and, after a cluster barrier,
// rank r reduces rows r, r+CS, ... over DSMEM summing the splits in global
// order (z = p0 + p1 + ... + b0).  CS is chosen per pack for occupancy
// (CS = nsplit is the one-split-per-CTA cluster forward; small CS streams);
// the arithmetic never depends on it, so packed == standalone bitwise.
__host__ __device__ inline int m1c_raw_stages(int RP) { return RP >= 128 ? 2 : 4; }
__host__ __device__ inline int m1c_region_floats(int RP) {  // raw ring + hi/lo buffers
  return m1c_raw_stages(RP) * (T_SC * T_UM + RP * T_SXLD) + 2 * 2 * (T_UM + RP) * T_SC;
}
__host__ __device__ inline int m1c_fwd_smem(int RP, int C) {
  return m1c_region_floats(RP) * 4 + T_UM * C * 4 + T_UM * 4 + RP * 4 + 2 * T_MAXCS * 4 + 64;
}
// most splits a CTA may own: TMEM columns and the partial + row buffers
__host__ __device__ inline int m1c_max_local(int RP) {
  const int by_tmem = 512 / RP;
  const int by_smem = (m1c_region_floats(RP) - RP * T_UM) / (RP * T_UM);
  return by_tmem < by_smem ? by_tmem : by_smem;
}
__host__ __device__ inline void m1c_range(int nsplit, int CS, int r, int* s0, int* n) {
  const int base = nsplit / CS, extra = nsplit % CS;
  *n = base + (r < extra ? 1 : 0);
  *s0 = r * base + (r < extra ? r : extra);
}

__device__ void m1c_fwd_tile(char* sm, const MemberDev<float>& M, const FeedDev<float>& f,
                             int tile, int rank, int CS, const PhaseArgs<float>& P) {
  const int D = M.dims[0], H = M.dims[1], C = M.dims[2];
  const int R = f.take, RP = m1_rows_pad(M.max_rows), S = m1c_raw_stages(RP);
  const int u0 = tile * T_UM, nu = min(T_UM, H - u0), nu4 = (nu + 3) & ~3;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nsplit = t_nsplit(D);
  int sbeg, nloc;
  m1c_range(nsplit, CS, rank, &sbeg, &nloc);
  const int c_beg = 2 * sbeg, c_end = min(2 * (sbeg + nloc), (D + T_SC - 1) / T_SC);
  const int nchl = c_end - c_beg;  // my chunks
  const int RSF = T_SC * T_UM + RP * T_SXLD;
  float* raw = reinterpret_cast<float*>(sm);
  float* hl = raw + S * RSF;
  const int HLF = 2 * (T_UM + RP) * T_SC;
  float* sW1 = raw + m1c_region_floats(RP);
  float* sb0 = sW1 + T_UM * C;
  int32_t* srow = reinterpret_cast<int32_t*>(sb0 + T_UM);
  int32_t* s_own = srow + RP;          // [T_MAXCS] owner rank of split s
  int32_t* s_loc = s_own + T_MAXCS;    // [T_MAXCS] local index within the owner
  uint64_t* bar = reinterpret_cast<uint64_t*>(s_loc + T_MAXCS);  // [0,1] full [2,3] empty [4] done
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 5);
  float* sP = raw;                      // after the loop: [nloc][RP][T_UM] partials
  float* sA = raw + nloc * RP * T_UM;   // then my rows' activations [nr][T_UM]
  const uint32_t tcols = umma::tmem_cols_pow2(max(nloc, 1) * RP);

  for (int r = tid; r < RP; r += NT) srow[r] = r < R ? (int32_t)feed_row(f, r) : 0;
  if (tid < CS) {
    int b0, n0;
    m1c_range(nsplit, CS, tid, &b0, &n0);
    for (int i = 0; i < n0; ++i) {
      s_own[b0 + i] = tid;
      s_loc[b0 + i] = i;
    }
  }
  if (tid == 32) {
    umma::mbar_init(&bar[0], 7);
    umma::mbar_init(&bar[1], 7);
    umma::mbar_init(&bar[2], 1);
    umma::mbar_init(&bar[3], 1);
    umma::mbar_init(&bar[4], 1);
    umma::mbar_fence_init();
  }
  if (warp == 1) umma::tmem_alloc(tslot, tcols);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = *tslot;
  // the member's state only after the previous step of a multi-step graph
  if (P.first) {
    pdl_wait();
    pdl_launch();
  }
  if (halted(P)) {  // uniform over the grid: no cluster barrier is left waiting
    umma::fence_before();
    __syncthreads();
    if (warp == 1) umma::tmem_dealloc(tmem, tcols);
    return;
  }
  const float* Pc = M.params[M.ctl->parity];
  const float* W0 = Pc + M.w_off[0];
  bool badx = false;
  if (warp < 7) {
    // ------------------------------------------------------------ producers
    const int pt = tid;
    auto issue = [&](int i) {  // my chunk i (global chunk c_beg + i) → stage i % S
      float* rA = raw + (i % S) * RSF;
      float* rX = rA + T_SC * T_UM;
      const int k0 = (c_beg + i) * T_SC, nk = min(T_SC, D - k0), cpr = nu4 / 4;
      for (int e = pt; e < nk * cpr; e += T_WS_PRODUCERS) {
        int k, q;
      divmod_p2(e, cpr, k, q);
        cp_async<16>(rA + k * T_UM + 4 * q, W0 + (int64_t)(k0 + k) * H + u0 + 4 * q, true);
      }
      const int cx = nk / 4;
      for (int e = pt; e < R * cx; e += T_WS_PRODUCERS) {
        int r, q;
      divmod_p2(e, cx, r, q);
        cp_async<16>(rX + r * T_SXLD + 4 * q, f.feat + (int64_t)srow[r] * f.ld + k0 + 4 * q, true);
      }
      cp_commit();
    };
    for (int e = pt; e < nu4 * C / 4; e += T_WS_PRODUCERS)
      cp_async<16>(sW1 + 4 * e, Pc + M.w_off[1] + (int64_t)u0 * C + 4 * e, true);
    for (int e = pt; e < nu4 / 4; e += T_WS_PRODUCERS)
      cp_async<16>(sb0 + 4 * e, Pc + M.b_off[0] + u0 + 4 * e, true);
    for (int i = 0; i < S - 1; ++i) {
      if (i < nchl) issue(i);
      else cp_commit();
    }
    uint32_t eph[2] = {0u, 0u};
    for (int i = 0; i < nchl; ++i) {
      if (i + S - 1 < nchl) issue(i + S - 1);
      else cp_commit();
      if (S == 4) cp_wait<3>(); else cp_wait<1>();
      asm volatile("bar.sync 1, %0;" ::"n"(T_WS_PRODUCERS) : "memory");  // chunk i landed
      const int b = i & 1;
      if (i >= 2) {
        umma::mbar_wait(&bar[2 + b], eph[b]);
        eph[b] ^= 1u;
      }
      float* Ah = hl + b * HLF;
      float* Al = Ah + T_UM * T_SC;
      float* Bh = Al + T_UM * T_SC;
      float* Bl = Bh + RP * T_SC;
      const float* rA = raw + (i % S) * RSF;
      const float* rX = rA + T_SC * T_UM;
      const int nk = min(T_SC, D - (c_beg + i) * T_SC);
      for (int e = pt; e < T_UM * (T_SC / 4); e += T_WS_PRODUCERS) {
        const int u = e % T_UM, kq = e / T_UM;
        float4 h, l;
        float* hp = &h.x;
        float* lp = &l.x;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int k = 4 * kq + j;
          const float v = (u < nu && k < nk) ? rA[k * T_UM + u] : 0.f;
          umma::split3(v, hp[j], lp[j]);
        }
        const uint32_t o = umma::kmaj_off(u, 4 * kq, T_UM) / 4;
        *reinterpret_cast<float4*>(Ah + o) = h;
        *reinterpret_cast<float4*>(Al + o) = l;
      }
      for (int e = pt; e < RP * (T_SC / 4); e += T_WS_PRODUCERS) {
        const int r = e % RP, kq = e / RP;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (r < R && 4 * kq < nk) v = *reinterpret_cast<const float4*>(rX + r * T_SXLD + 4 * kq);
        badx |= !finite(v.x) | !finite(v.y) | !finite(v.z) | !finite(v.w);
        float4 h, l;
        umma::split3(v.x, h.x, l.x);
        umma::split3(v.y, h.y, l.y);
        umma::split3(v.z, h.z, l.z);
        umma::split3(v.w, h.w, l.w);
        const uint32_t o = umma::kmaj_off(r, 4 * kq, RP) / 4;
        *reinterpret_cast<float4*>(Bh + o) = h;
        *reinterpret_cast<float4*>(Bl + o) = l;
      }
      umma::fence_async_smem();
      asm volatile("bar.sync 1, %0;" ::"n"(T_WS_PRODUCERS) : "memory");
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(umma::smem_u32(&bar[b]))
                     : "memory");
    }
    cp_wait<0>();
  } else if (lane == 0) {
    // --------------------------------------------------------- MMA issuer
    const uint32_t idesc = umma::idesc_tf32(T_UM, RP, false, false);
    uint32_t fph[2] = {0u, 0u};
    for (int i = 0; i < nchl; ++i) {
      const int b = i & 1, c = c_beg + i;
      umma::mbar_wait(&bar[b], fph[b]);
      fph[b] ^= 1u;
      umma::fence_after();
      float* Ah = hl + b * HLF;
      float* Al = Ah + T_UM * T_SC;
      float* Bh = Al + T_UM * T_SC;
      float* Bl = Bh + RP * T_SC;
      const uint32_t ah = umma::smem_u32(Ah), al = umma::smem_u32(Al);
      const uint32_t bh = umma::smem_u32(Bh), bl = umma::smem_u32(Bl);
      const uint32_t acc = tmem + (uint32_t)(((c >> 1) - sbeg) * RP);
      const int nk = min(T_SC, D - c * T_SC);
      for (int s2 = 0; s2 < (nk + 7) / 8; ++s2) {
        const uint64_t dah = umma::kmaj_desc(ah, T_UM, s2), dal = umma::kmaj_desc(al, T_UM, s2);
        const uint64_t dbh = umma::kmaj_desc(bh, RP, s2), dbl = umma::kmaj_desc(bl, RP, s2);
        umma::mma_tf32(acc, dah, dbh, idesc, (c & 1) || s2 > 0);
        umma::mma_tf32(acc, dah, dbl, idesc, true);
        umma::mma_tf32(acc, dal, dbh, idesc, true);
      }
      umma::commit(&bar[2 + b]);
    }
    umma::commit(&bar[4]);
  }
  umma::mbar_wait(&bar[4], 0);
  umma::fence_after();
  badx = __syncthreads_or(badx);  // also: the raw / hi-lo region is free
  if (badx && tid == 0) flag_min(&M.ctl->bad_node, 0);
  PK_TRACE(2);
  // ---- my split partials: TMEM → sP[local][r][u] ----------------------------
  {
    const int q = warp & 3, half = warp >> 2, u = 32 * q + lane;
    for (int l = 0; l < nloc; ++l)
      for (int c0 = half * (RP / 2); c0 < (half + 1) * (RP / 2); c0 += 8) {
        float v[8];
        umma::tmem_ld8(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(l * RP + c0), v);
        umma::tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 8; ++i) sP[(l * RP + c0 + i) * T_UM + u] = v[i];
      }
  }
  umma::fence_before();
  umma::cluster_sync();  // every split's partial is in the cluster's shared memory
  PK_TRACE(3);
  if (warp == 1) umma::tmem_dealloc(tmem, tcols);
  // ---- rank r reduces rows r, r + CS, ...: z = Σ_s p_s in split order ------
  const int nr = R > rank ? (R - rank + CS - 1) / CS : 0;
  int bad = INT_MAX;
  // four consecutive units per thread: one 16-byte DSMEM load per split
  for (int e4 = tid; e4 < nr * T_UM / 4; e4 += NT) {
    const int rl = e4 / (T_UM / 4), u = 4 * (e4 % (T_UM / 4)), r = rank + rl * CS;
    float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    if (u < nu) {
      float4 v[T_MAXCS];
#pragma unroll
      for (int sp = 0; sp < T_MAXCS; ++sp)
        v[sp] = sp < nsplit
                    ? umma::dsmem_ld4(umma::smem_u32(sP + (s_loc[sp] * RP + r) * T_UM + u),
                                      (uint32_t)s_own[sp])
                    : make_float4(0.f, 0.f, 0.f, 0.f);
      z = v[0];
#pragma unroll
      for (int sp = 1; sp < T_MAXCS; ++sp)
        if (sp < nsplit) {
          z.x += v[sp].x;
          z.y += v[sp].y;
          z.z += v[sp].z;
          z.w += v[sp].w;
        }
    }
    m1_finish4(M, z, sb0, r, u, R, nu, u0, H, sA + rl * T_UM + u, &bad);
  }
  __syncthreads();
  const int nbt = (nu + T_LB - 1) / T_LB;
  for (int e = tid; e < nbt * nr * C; e += NT) {
    const int bl = e / (nr * C), rc = e % (nr * C), rl = rc / C, c = rc % C;
    const int ub = bl * T_LB, r = rank + rl * CS;
    const float* a = sA + rl * T_UM + ub;
    const float* w = sW1 + ub * C + c;
    float p = 0.f;
#pragma unroll 8
    for (int j = 0; j < T_LB; ++j) p = fmaf(a[j], ub + j < nu ? w[j * C] : 0.f, p);
    M.Z[1][((int64_t)(u0 / T_LB + bl) * M.max_rows + r) * C + c] = p;
  }
  if (bad != INT_MAX) flag_min(&M.ctl->bad_node, bad);
  PK_TRACE(4);
  umma::cluster_arrive_relaxed();  // peers are done reading this CTA's partials
  umma::cluster_wait();
}

// ----------------------------------------------------------- backward --
// One CTA per (member, 32-unit tile, group of `ng` consecutive 128-input
// tiles).  The per-unit-tile work — logits, softmax-xent, dZ0 — is done once
// and the group's W0 tiles (+ slots, + X columns) stream through S shared-
// memory stages by 16-byte cp.async while the previous tile's MMA and optimizer
// epilogue run.  Which CTA updates an element never changes its arithmetic,
// so the grouping (chosen per pack for occupancy) keeps K-invariance.
// The tensor / cluster paths' optimizer on one fp32 element (engine.py:302-324).
// Every operation is an explicit round-to-nearest intrinsic: no FMA
// contraction, so the update is bit-identical in every kernel and template
// instantiation that applies it (packed == standalone does not depend on how
// the compiler scheduled a particular copy).  ib1 / ib2 = 1 / Adam's bias
// corrections (≤ 1 ulp from the divisions; the fp32 contract is rel 1e-4).
// the MUFU square root and reciprocal (≤ 2 ulp): one instruction each
// instead of the IEEE-exact sequences, deterministic in every kernel copy;
// the fp32 contract is rel 1e-4
__device__ __forceinline__ float sqrt_mufu(float x) {
  float r;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rcp_mufu(float x) {
  float r;
  asm("rcp.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ void opt_x(int opt, float lr, float wd, float ib1, float ib2, float& w,
                                      float& s0, float& s1, float g) {
  if (wd != 0.f) g = __fadd_rn(g, __fmul_rn(wd, w));
  switch (opt) {
    case PK_OPT_SGD:
      w = __fsub_rn(w, __fmul_rn(lr, g));
      break;
    case PK_OPT_MOMENTUM:
      s0 = __fadd_rn(__fmul_rn(s0, 0.9f), g);
      w = __fsub_rn(w, __fmul_rn(lr, s0));
      break;
    case PK_OPT_ADAGRAD:
      s0 = __fadd_rn(s0, __fmul_rn(g, g));
      w = __fsub_rn(w, __fmul_rn(__fmul_rn(lr, g), rcp_mufu(__fadd_rn(sqrt_mufu(s0), 1e-10f))));
      break;
    default:
      s0 = __fadd_rn(__fmul_rn(s0, 0.9f), __fmul_rn(1.f - 0.9f, g));
      s1 = __fadd_rn(__fmul_rn(s1, 0.999f), __fmul_rn(__fmul_rn(1.f - 0.999f, g), g));
      w = __fsub_rn(w, __fmul_rn(__fmul_rn(lr, __fmul_rn(s0, ib1)),
                                 rcp_mufu(__fadd_rn(sqrt_mufu(__fmul_rn(s1, ib2)), 1e-8f))));
      break;
  }
}

// 256-bit global accesses (sm_100): one full 32-byte sector per lane
__device__ __forceinline__ void ld8g(const float* p, float4& a, float4& b) {
  asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z),
                 "=f"(b.w)
               : "l"(p));
}
__device__ __forceinline__ void st8g(float* p, float4 a, float4 b) {
  asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(a.x), "f"(a.y),
               "f"(a.z), "f"(a.w), "f"(b.x), "f"(b.y), "f"(b.z), "f"(b.w)
               : "memory");
}

// the member's optimizer on four elements; ib1 / ib2 = 1 / Adam's bias
// corrections, computed once per tile by the caller (opt_recips)
__device__ __forceinline__ void opt_step4(int opt, float lr, float wd, float ib1, float ib2,
                                          float4& w, float4& s0, float4& s1, float4 g) {
  opt_x(opt, lr, wd, ib1, ib2, w.x, s0.x, s1.x, g.x);
  opt_x(opt, lr, wd, ib1, ib2, w.y, s0.y, s1.y, g.y);
  opt_x(opt, lr, wd, ib1, ib2, w.z, s0.z, s1.z, g.z);
  opt_x(opt, lr, wd, ib1, ib2, w.w, s0.w, s1.w, g.w);
}

// scalar form for the small W1 / b0 / b1 updates
__device__ __forceinline__ void opt_step1(int opt, float lr, float wd, float ib1, float ib2,
                                          float& w, float& s0, float& s1, float g) {
  opt_x(opt, lr, wd, ib1, ib2, w, s0, s1, g);
}

// Adam's bias-correction reciprocals 1/(1-β^t) of the member's control block
// (1 for the other optimizers)
__device__ __forceinline__ void opt_recips(int opt, const MemberCtl* ctl, float* ib1, float* ib2) {
  *ib1 = opt == PK_OPT_ADAM ? 1.f / float(ctl->bc1) : 1.f;
  *ib2 = opt == PK_OPT_ADAM ? 1.f / float(ctl->bc2) : 1.f;
}

// A operand of the weight-gradient MMA: Xᵀ rows k (128) × K = batch rows
// r0..r0+31, tf32 hi/lo, K-major; zero outside the valid box
__device__ __forceinline__ void m1t_stage_xT(float* Ah, float* Al, const float* sX, int r0, int R,
                                             int nk, int nthreads) {
  for (int e = threadIdx.x; e < T_BK * 8; e += nthreads) {
    const int k = e % T_BK, rq = e / T_BK;
    float4 h, l;
    float* hp = &h.x;
    float* lp = &l.x;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = r0 + 4 * rq + j;
      const float v = (r < R && k < nk) ? sX[r * T_BXLD + k] : 0.f;
      umma::split3(v, hp[j], lp[j]);
    }
    const uint32_t o = umma::kmaj_off(k, 4 * rq, T_BK) / 4;
    *reinterpret_cast<float4*>(Ah + o) = h;
    *reinterpret_cast<float4*>(Al + o) = l;
  }
}

__device__ __forceinline__ int m1t_bwd_stage_floats(int RP, int ns) {
  return T_BK * T_BWLD + RP * T_BXLD;  // W0 tile + X columns
}

__device__ __forceinline__ void cp_wait_n(int n) {  // pending commit groups allowed (<= 4)
  // predicated waits, no branch: a switch here compiles to a jump table
  // (LDC + BRX) whose indirect fetch costs hundreds of cycles per call
  asm volatile(
      "{\n\t.reg .pred p0, p1, p2, p3, p4;\n\t"
      "setp.le.s32 p0, %0, 0;\n\tsetp.eq.s32 p1, %0, 1;\n\tsetp.eq.s32 p2, %0, 2;\n\t"
      "setp.eq.s32 p3, %0, 3;\n\tsetp.ge.s32 p4, %0, 4;\n\t"
      "@p0 cp.async.wait_group 0;\n\t@p1 cp.async.wait_group 1;\n\t"
      "@p2 cp.async.wait_group 2;\n\t@p3 cp.async.wait_group 3;\n\t"
      "@p4 cp.async.wait_group 4;\n\t}\n" ::"r"(n)
      : "memory");
}

__device__ void m1t_bwd_tile(char* sm, const MemberDev<float>& M, const FeedDev<float>& f,
                             int kt0, int ng, int utile, int S_launch, int G) {
  const int D = M.dims[0], H = M.dims[1], C = M.dims[2];
  const int R = f.take, RP = m1_rows_pad(M.max_rows), ns = M.n_slots;
  // input-tile stages: as many as this member's shapes leave room for in the
  // launch's dynamic shared memory (the pack's largest member sets it), 1..4
  uint32_t dyn;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
  const int S = max(1, min(4, ((int)dyn - M1T::bwd_smem(RP, C, ns, 0)) /
                                  (4 * m1t_bwd_stage_floats(RP, ns))));
  (void)S_launch;
  const int u0 = utile * T_BU, nu = min(T_BU, H - u0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int BT = T_BWD_NT;  // this kernel runs 12 warps
  const MemberCtl* ctl = M.ctl;
  const int par = ctl->parity;
  const int64_t NP = M.s_stride;  // slot block stride (16-byte multiple)
  const float* __restrict__ Pc = M.params[par];
  float* __restrict__ Pn = M.params[par ^ 1];
  const float* __restrict__ Sc = M.slots[par];
  float* __restrict__ Sn = M.slots[par ^ 1];
  // smem carve: S stages of {W0 tile + slots [1+ns][T_BK][T_BU], X columns [RP][T_BXLD]}
  float* stg = reinterpret_cast<float*>(sm);
  const int SF = m1t_bwd_stage_floats(RP, ns);
  float* Ah = stg + S * SF;                             // K-major [8][T_BK][4]
  float* Al = Ah + T_BK * 32;
  float* Bh = Al + T_BK * 32;                           // K-major [8][T_BU][4]
  float* Bl = Bh + T_BU * 32;
  float* sL = Bl + T_BU * 32;                           // [RP][T_MAXC+1]
  const int LDL = C + 1;                                // sL row stride
  float* sdZ = sL + RP * LDL;                           // [RP][T_BU]
  float* sA0 = sdZ + RP * T_BU;                         // [RP][T_BU] A0 tile
  float* sW1 = sA0 + RP * T_BU;                         // [1+ns][T_BU][C]
  float* sb1 = sW1 + (1 + ns) * T_BU * C;               // [T_MAXC]
  int32_t* srow = reinterpret_cast<int32_t*>(sb1 + T_MAXC);
  int32_t* ylab = srow + RP;
  uint64_t* bar = reinterpret_cast<uint64_t*>(ylab + RP);  // [3] unused, [4..13] pipeline
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 14);
  constexpr uint32_t tcols = 64;  // two 32-column gradient buffers

  // ---- prologue (independent of k_m1t_fwd) --------------------------------
  for (int r = tid; r < RP; r += BT) {
    srow[r] = r < R ? (int32_t)feed_row(f, r) : 0;
    ylab[r] = r < R ? f.labels[feed_row(f, r)] : 0;
  }
  for (int c = tid; c < C; c += BT) sb1[c] = Pc[M.b_off[1] + c];
  if (warp == 0) umma::tmem_alloc(tslot, tcols);
  if (tid == 32) {
    umma::mbar_init(&bar[3], 1);
    umma::mbar_fence_init();
  }
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = *tslot;
  // 16-byte cp.async (LDGSTS) from every thread; one commit group per input
  // tile, staged into stage i % S
  auto issue = [&](int i) {
    const int k0 = (kt0 + i) * T_BK, nk = min(T_BK, D - k0);
    float* sW = stg + (i % S) * SF;
    float* sX = sW + T_BK * T_BWLD;
    const int cw = nu / 4, cx = nk / 4;
    {
      const float* src = Pc + M.w_off[0] + u0;
      for (int e = tid; e < nk * cw; e += BT) {
        int k, c;
        divmod_p2(e, cw, k, c);
        cp_async<16>(sW + k * T_BWLD + 4 * c, src + (int64_t)(k0 + k) * H + 4 * c, true);
      }
    }
    for (int e = tid; e < R * cx; e += BT) {
      int r, c;
      divmod_p2(e, cx, r, c);
      cp_async<16>(sX + r * T_BXLD + 4 * c, f.feat + (int64_t)srow[r] * f.ld + k0 + 4 * c, true);
    }
    cp_commit();
  };
  for (int s = 0; s <= ns; ++s) {  // W1 rows (+ slots): the first commit group
    const float* src = (s == 0 ? Pc : Sc + (int64_t)(s - 1) * NP) + M.w_off[1] + (int64_t)u0 * C;
    for (int e = tid; e < nu * C / 4; e += BT) cp_async<16>(sW1 + s * T_BU * C + 4 * e, src + 4 * e, true);
  }
  cp_commit();
  const int nstg = min(S, ng);
  for (int i = 0; i < nstg; ++i) issue(i);
  const int nch = RP / 32;
  // A = X[:, tile 0]ᵀ (hi/lo) does not depend on the forward: stage it now,
  // overlapping k_m1t_fwd, when one 32-row chunk covers the batch
  const bool a_ready = nch == 1;
  if (a_ready) {
    cp_wait_n(nstg - 1);  // stage 0 landed
    __syncthreads();
    m1t_stage_xT(Ah, Al, stg + T_BK * T_BWLD, 0, R, min(T_BK, D - kt0 * T_BK), BT);
  }
  pdl_wait();  // k_m1t_fwd's Z0 / A0 / partial logits are visible
  PK_TRACE(1);
  // Z0 / A0 of the tile's units (dZ0 below) do not depend on the logits: their
  // loads fly while the logits are summed and the softmax-xent runs
  constexpr int PER = (T_MAXR * T_BU + BT - 1) / BT;  // elements per thread
  float zr[PER], ar[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int e = tid + i * BT, r = e / T_BU, j = e % T_BU;
    const bool ok = e < RP * T_BU && r < R && j < nu;
    const int64_t g = (int64_t)r * H + u0 + j;
    zr[i] = ok ? M.Z[0][g] : 0.f;
    ar[i] = ok ? M.A[0][g] : 0.f;
  }
  // ---- logits = Σ_blk partials + b1 → softmax-xent → dZ1 (in sL) ----------
  const int nb = t_nblk(H);
  const bool owner = (kt0 == 0 && utile == 0);
  int bad = INT_MAX;
  const int64_t bstr = (int64_t)M.max_rows * C;
  for (int e = tid; e < R * C; e += BT) {
    const int c = e % C;
    const float* pp = M.Z[1] + e;
    float z = 0.f;
    for (int q0 = 0; q0 < nb; q0 += 8) {  // block partials in flight, summed in block order
      float v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = q0 + j < nb ? pp[(q0 + j) * bstr] : 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (q0 + j < nb) z = (q0 + j == 0) ? v[j] : z + v[j];
    }
    const int r = e / C;
    z += sb1[c];
    sL[r * LDL + c] = z;
    if (!finite(z)) bad = 3;
  }
  if (owner && bad != INT_MAX) flag_min(&M.ctl->bad_node, bad);
  __syncthreads();
  PK_TRACE(8);
  for (int r0 = 0; r0 < R; r0 += BT / 8) {  // 8 lanes per row, every warp busy
    const int r = r0 + (tid >> 3);
    xent_row8(sL + min(r, R - 1) * LDL, C, ylab[min(r, R - 1)], R, r < R,
              owner && r < R ? M.rowloss + r : nullptr);
  }
  PK_TRACE(9);
  cp_wait_n(nstg);  // W1 rows (the first group) landed
  __syncthreads();
  PK_TRACE(10);
  if (owner && warp == 0) {
    // the member's step loss (finalize's lane-strided order) and Adam's bias
    // corrections for the *next* update, off finalize's serial tail
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
  // ---- dZ0[:, units] = (dZ1 · W1[units, :]ᵀ) ⊙ act'(Z0, A0) ----------------
  {
#pragma unroll
    for (int i = 0; i < PER; ++i) {  // park Z0 / A0 in shared memory (own elements)
      const int e = tid + i * BT;
      if (e < RP * T_BU) {
        sdZ[e] = zr[i];
        sA0[e] = ar[i];
      }
    }
#pragma unroll 1
    for (int e = tid; e < RP * T_BU; e += BT) {  // one rolled body, one act' switch
      const int r = e / T_BU, j = e % T_BU;
      float v = 0.f;
      if (r < R && j < nu) {
        float s = 0.f;
        for (int c = 0; c < C; ++c) s = fmaf(sL[r * LDL + c], sW1[j * C + c], s);
        v = act_bwd(M.act, sdZ[e], sA0[e], s);
      }
      sdZ[e] = v;
    }
  }
  __syncthreads();
  PK_TRACE(11);
  const float lr = float(ctl->lr), wd = float(M.wd);
  float bc1, bc2;  // (reciprocals)
  opt_recips(M.opt, ctl, &bc1, &bc2);
  const int fault = ctl->fault_grad;
  bool badW0 = false, badW1 = false, badb1 = false, badb0 = false;
  // ---- stream the group's input tiles, warp-specialised -------------------
  //   warps 0-7 (epilogue): TMEM gradient → optimizer against the resident W0
  //                         tile → Pn/Sn; frees the TMEM buffer and the stage
  //   warps 8-10 (producers): Xᵀ / dZ0 hi-lo staging per 32-row chunk, the
  //                         cp.async of the next input tile
  //   warp 11 lane 0 (MMA): 12 tcgen05.mma per chunk into TMEM buffer i & 1
  // so tile i's optimizer epilogue overlaps tile i+1's staging and MMAs.
  // mbarriers: 4 afull (count 3), 5 aempty, 6/7 tfull, 8/9 tempty (count 8),
  // 10/11 sfree (count 8)
  const uint32_t idesc = umma::idesc_tf32(T_BK, T_BU, false, false);
  cp_wait<0>();  // the prologue's stages (issued by every thread) have landed
  if (tid == 32) {
    umma::mbar_init(&bar[4], 3);
    umma::mbar_init(&bar[5], 1);
    for (int j = 6; j < 10; ++j) umma::mbar_init(&bar[j], j < 8 ? 1 : 8);
    for (int j = 10; j < 14; ++j) umma::mbar_init(&bar[j], 8);
    umma::mbar_fence_init();
  }
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  if (warp < 8) {
    // -------------------------------------------------------------- epilogue
    // ---- W1[units, :] (grad 0), b1 (grad 1), b0[units] (grad 3), element e
    //      of the unit tile by the tile's group gi ≡ e (mod ngr): done here,
    //      while the producers stage and the MMA warp multiplies tile 0
    {
      const int gi = kt0 / G, ngr = (cdiv_d(D, T_BK) + G - 1) / G;
      for (int e = gi + ngr * tid; e < nu * C; e += ngr * 256) {
        const int j = e / C, c = e % C;
        float g = 0.f;
        for (int r = 0; r < R; ++r) g = fmaf(sA0[r * T_BU + j], sL[r * LDL + c], g);
        if (fault == 0) g = NAN;
        badW1 |= !finite(g);
        float w = sW1[e], s0 = ns >= 1 ? sW1[T_BU * C + e] : 0.f,
              s1 = ns >= 2 ? sW1[2 * T_BU * C + e] : 0.f;
        opt_step1(M.opt, lr, wd, bc1, bc2, w, s0, s1, g);
        const int64_t i = M.w_off[1] + (int64_t)u0 * C + e;
        Pn[i] = w;
        if (ns >= 1) Sn[i] = s0;
        if (ns >= 2) Sn[NP + i] = s1;
      }
      if (utile == 0) {
        for (int c = gi + ngr * tid; c < C; c += ngr * 256) {
          float g = 0.f;
          for (int r = 0; r < R; ++r) g += sL[r * LDL + c];
          if (fault == 1) g = NAN;
          badb1 |= !finite(g);
          const int64_t i = M.b_off[1] + c;
          float w = Pc[i], s0 = ns >= 1 ? Sc[i] : 0.f, s1 = ns >= 2 ? Sc[NP + i] : 0.f;
          opt_step1(M.opt, lr, wd, bc1, bc2, w, s0, s1, g);
          Pn[i] = w;
          if (ns >= 1) Sn[i] = s0;
          if (ns >= 2) Sn[NP + i] = s1;
        }
      }
      for (int j = gi + ngr * tid; j < nu; j += ngr * 256) {
        float g = 0.f;
        for (int r = 0; r < R; ++r) g += sdZ[r * T_BU + j];
        if (fault == 3) g = NAN;
        badb0 |= !finite(g);
        const int64_t i = M.b_off[0] + u0 + j;
        float w = Pc[i], s0 = ns >= 1 ? Sc[i] : 0.f, s1 = ns >= 2 ? Sc[NP + i] : 0.f;
        opt_step1(M.opt, lr, wd, bc1, bc2, w, s0, s1, g);
        Pn[i] = w;
        if (ns >= 1) Sn[i] = s0;
        if (ns >= 2) Sn[NP + i] = s1;
      }
    }
    // warp w: TMEM lane quarter w % 4 (input rows k), column half w / 4
    const int k = 32 * (warp & 3) + lane, ch16 = (warp >> 2) * 16;
    // full 16-unit halves on 32-byte boundaries: 256-bit slot / param I/O
    const bool wide8 = H % 8 == 0 && NP % 8 == 0 && u0 % 8 == 0 && ch16 + 16 <= nu;
    for (int i = 0; i < ng; ++i) {
      const int t = i & 1, st = i % S;
      const int k0 = (kt0 + i) * T_BK, nk = min(T_BK, D - k0);
      // optimizer slots of my 16 elements straight from global memory, in
      // flight while the tile's MMAs finish (the stages hold only W0 + X)
      float4 sl0[4], sl1[4];
      {
        const int64_t ib = M.w_off[0] + (int64_t)(k0 + min(k, nk - 1)) * H + u0 + ch16;
        if (wide8 && k < nk) {  // two 256-bit loads per slot block
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (ns >= 1) ld8g(Sc + ib + 8 * h, sl0[2 * h], sl0[2 * h + 1]);
            else sl0[2 * h] = sl0[2 * h + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (ns >= 2) ld8g(Sc + NP + ib + 8 * h, sl1[2 * h], sl1[2 * h + 1]);
            else sl1[2 * h] = sl1[2 * h + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        } else {
#pragma unroll
          for (int qd = 0; qd < 4; ++qd) {
            const bool ok = k < nk && ch16 + 4 * qd < nu;
            sl0[qd] = ns >= 1 && ok ? *reinterpret_cast<const float4*>(Sc + ib + 4 * qd)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
            sl1[qd] = ns >= 2 && ok ? *reinterpret_cast<const float4*>(Sc + NP + ib + 4 * qd)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
      }
      umma::mbar_wait(&bar[6 + t], (uint32_t)((i >> 1) & 1));
      umma::fence_after();
      float g[16];
#pragma unroll
      for (int c8 = 0; c8 < 2; ++c8) {
        float v[8];
        umma::tmem_ld8(tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(t * T_BU + ch16 + 8 * c8), v);
#pragma unroll
        for (int j = 0; j < 8; ++j) g[8 * c8 + j] = v[j];
      }
      umma::tmem_wait_ld();
      umma::fence_before();
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(umma::smem_u32(&bar[8 + t]))
                     : "memory");
      if (i == min(1, ng - 1)) PK_TRACE(14);
      const float* sW = stg + st * SF;
      if (k < nk && wide8) {
        // 16 units of one row: two pairs of quads, each written as one
        // 256-bit store per stream (full sectors, half the transactions)
        const int64_t i0 = M.w_off[0] + (int64_t)(k0 + k) * H + u0 + ch16;
        const float* row = sW + k * T_BWLD + ch16;
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          float4 gq[2], w[2], s0[2], s1[2];
          if (h == 0) {
            gq[0] = make_float4(g[0], g[1], g[2], g[3]);
            gq[1] = make_float4(g[4], g[5], g[6], g[7]);
            s0[0] = sl0[0]; s0[1] = sl0[1]; s1[0] = sl1[0]; s1[1] = sl1[1];
          } else {
            gq[0] = make_float4(g[8], g[9], g[10], g[11]);
            gq[1] = make_float4(g[12], g[13], g[14], g[15]);
            s0[0] = sl0[2]; s0[1] = sl0[3]; s1[0] = sl1[2]; s1[1] = sl1[3];
          }
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            if (fault == 2) gq[j] = make_float4(NAN, NAN, NAN, NAN);
            badW0 |= !finite(gq[j].x) | !finite(gq[j].y) | !finite(gq[j].z) | !finite(gq[j].w);
            w[j] = *reinterpret_cast<const float4*>(row + 8 * h + 4 * j);
            opt_step4(M.opt, lr, wd, bc1, bc2, w[j], s0[j], s1[j], gq[j]);
          }
          st8g(Pn + i0 + 8 * h, w[0], w[1]);
          if (ns >= 1) st8g(Sn + i0 + 8 * h, s0[0], s0[1]);
          if (ns >= 2) st8g(Sn + NP + i0 + 8 * h, s1[0], s1[1]);
        }
      } else if (k < nk) {
        const int64_t i0 = M.w_off[0] + (int64_t)(k0 + k) * H + u0 + ch16;
        const float* row = sW + k * T_BWLD + ch16;
        // one rolled quad loop, one optimizer body (nu % 4 == 0)
#pragma unroll 1
        for (int qd = 0; qd < 4; ++qd) {
          if (ch16 + 4 * qd >= nu) break;
          float4 gq, s0, s1;
          switch (qd) {  // registers cannot be indexed dynamically: select
            case 0: gq = make_float4(g[0], g[1], g[2], g[3]); s0 = sl0[0]; s1 = sl1[0]; break;
            case 1: gq = make_float4(g[4], g[5], g[6], g[7]); s0 = sl0[1]; s1 = sl1[1]; break;
            case 2: gq = make_float4(g[8], g[9], g[10], g[11]); s0 = sl0[2]; s1 = sl1[2]; break;
            default: gq = make_float4(g[12], g[13], g[14], g[15]); s0 = sl0[3]; s1 = sl1[3]; break;
          }
          if (fault == 2) gq = make_float4(NAN, NAN, NAN, NAN);
          badW0 |= !finite(gq.x) | !finite(gq.y) | !finite(gq.z) | !finite(gq.w);
          float4 w = *reinterpret_cast<const float4*>(row + 4 * qd);
          opt_step4(M.opt, lr, wd, bc1, bc2, w, s0, s1, gq);
          *reinterpret_cast<float4*>(Pn + i0 + 4 * qd) = w;
          if (ns >= 1) *reinterpret_cast<float4*>(Sn + i0 + 4 * qd) = s0;
          if (ns >= 2) *reinterpret_cast<float4*>(Sn + NP + i0 + 4 * qd) = s1;
        }
      }
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(umma::smem_u32(&bar[10 + st]))
                     : "memory");
      if (i == min(1, ng - 1)) PK_TRACE(15);
    }
  } else if (warp < 11) {
    // ------------------------------------------------------------- producers
    const int pt = tid - 256;
    constexpr int NP3 = 96;
    auto issue_p = [&](int i) {  // input tile i of the group → stage i % S
      const int k0 = (kt0 + i) * T_BK, nk = min(T_BK, D - k0);
      float* sW = stg + (i % S) * SF;
      float* sX = sW + T_BK * T_BWLD;
      const int cw = nu / 4, cx = nk / 4;
      {
        const float* src = Pc + M.w_off[0] + u0;
        for (int e = pt; e < nk * cw; e += NP3) {
          int kk, c;
          divmod_p2(e, cw, kk, c);
          cp_async<16>(sW + kk * T_BWLD + 4 * c, src + (int64_t)(k0 + kk) * H + 4 * c, true);
        }
        // the epilogue reads this tile's optimizer slots from global: pull
        // them into L2 now, one line prefetch per row segment
        for (int e = pt; e < ns * nk; e += NP3) {
          const int s2 = e / nk, kk = e % nk;
          l2_prefetch_lines(Sc + (int64_t)s2 * NP + M.w_off[0] + (int64_t)(k0 + kk) * H + u0,
                            (uint32_t)(nu * 4));
        }
      }
      for (int e = pt; e < R * cx; e += NP3) {
        int r, c;
      divmod_p2(e, cx, r, c);
        cp_async<16>(sX + r * T_BXLD + 4 * c, f.feat + (int64_t)srow[r] * f.ld + k0 + 4 * c, true);
      }
      cp_commit();
    };
    uint32_t aph = 0;
    bool first = true;
    int next = min(S, ng);  // tiles [0, next) issued
    for (int i = 0; i < ng; ++i) {
      if (i >= S) {  // issued by the producers: wait for it (later groups may fly)
        cp_wait_n(next - 1 - i);
        asm volatile("bar.sync 2, 96;" ::: "memory");
      }
      const int nk = min(T_BK, D - (kt0 + i) * T_BK);
      const float* sX = stg + (i % S) * SF + T_BK * T_BWLD;
      for (int ch = 0; ch < nch; ++ch) {
        if (!first) {
          umma::mbar_wait(&bar[5], aph);
          aph ^= 1u;
        }
        first = false;
        if (!(a_ready && i == 0 && ch == 0)) {  // A = Xᵀ rows k, K = rows r
          for (int e = pt; e < T_BK * 8; e += NP3) {
            const int kk = e % T_BK, rq = e / T_BK;
            float4 h, l;
            float* hp = &h.x;
            float* lp = &l.x;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int r = ch * 32 + 4 * rq + j;
              const float v = (r < R && kk < nk) ? sX[r * T_BXLD + kk] : 0.f;
              umma::split3(v, hp[j], lp[j]);
            }
            const uint32_t o = umma::kmaj_off(kk, 4 * rq, T_BK) / 4;
            *reinterpret_cast<float4*>(Ah + o) = h;
            *reinterpret_cast<float4*>(Al + o) = l;
          }
        }
        for (int e = pt; e < T_BU * 8; e += NP3) {  // B = dZ0ᵀ rows u, K = rows r
          const int u = e % T_BU, rq = e / T_BU;
          float4 h, l;
          float* hp = &h.x;
          float* lp = &l.x;
#pragma unroll
          for (int j = 0; j < 4; ++j) umma::split3(sdZ[(ch * 32 + 4 * rq + j) * T_BU + u], hp[j], lp[j]);
          const uint32_t o = umma::kmaj_off(u, 4 * rq, T_BU) / 4;
          *reinterpret_cast<float4*>(Bh + o) = h;
          *reinterpret_cast<float4*>(Bl + o) = l;
        }
        umma::fence_async_smem();
        asm volatile("bar.sync 2, 96;" ::: "memory");
        if (lane == 0)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(umma::smem_u32(&bar[4]))
                       : "memory");
      }
      // refill: tile `next` reuses the stage of tile next - S once its
      // epilogue is done; with S >= 3 stay two epilogues behind (no stall)
      const int limit = S >= 3 ? i + S - 2 : i + 1;
      while (next < ng && next <= limit) {
        const int j = next - S;
        umma::mbar_wait(&bar[10 + (j % S)], (uint32_t)((j / S) & 1));
        issue_p(next);
        ++next;
      }
    }
    cp_wait<0>();
  } else if (lane == 0) {
    // ------------------------------------------------------------ MMA issuer
    uint32_t fph = 0;
    const uint32_t ah = umma::smem_u32(Ah), al = umma::smem_u32(Al);
    const uint32_t bh = umma::smem_u32(Bh), bl = umma::smem_u32(Bl);
    for (int i = 0; i < ng; ++i) {
      const int t = i & 1;
      if (i >= 2) umma::mbar_wait(&bar[8 + t], (uint32_t)(((i - 2) >> 1) & 1));
      for (int ch = 0; ch < nch; ++ch) {
        umma::mbar_wait(&bar[4], fph);
        fph ^= 1u;
        umma::fence_after();
        if (i == min(1, ng - 1) && ch == 0) PK_TRACE(13);
        const uint32_t acc = tmem + (uint32_t)(t * T_BU);
        for (int s2 = 0; s2 < 4; ++s2) {
          const uint64_t dah = umma::kmaj_desc(ah, T_BK, s2), dal = umma::kmaj_desc(al, T_BK, s2);
          const uint64_t dbh = umma::kmaj_desc(bh, T_BU, s2), dbl = umma::kmaj_desc(bl, T_BU, s2);
          umma::mma_tf32(acc, dah, dbh, idesc, ch > 0 || s2 > 0);
          umma::mma_tf32(acc, dah, dbl, idesc, true);
          umma::mma_tf32(acc, dal, dbh, idesc, true);
        }
        umma::commit(&bar[5]);  // A/B hi-lo buffers free
      }
      umma::commit(&bar[6 + t]);  // the tile's gradient is in TMEM buffer t
    }
  }
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  PK_TRACE(3);
  PK_TRACE(4);
  if (badW1) flag_min(&M.ctl->bad_grad, 0);
  if (badb1) flag_min(&M.ctl->bad_grad, 1);
  if (badW0) flag_min(&M.ctl->bad_grad, 2);
  if (badb0) flag_min(&M.ctl->bad_grad, 3);
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tmem, tcols);
}
