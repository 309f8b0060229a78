// Gram-path interpolative decomposition of large separators (included from kernels.cu: it
// reuses the chunked coupling-row gather, the ArgMax reduction and the DMMA helpers there).
//
// Reference: kernels.py:84-119 (ID by column-pivoted QR, dgeqp3) as restated in
// oracle/dense.py:cpqr_dlaqp2. CPQR pivots and |R_ii| depend on A only through the Gram
// matrix A^T A: the Householder step i turns column j's remaining part into one whose norm^2
// is the Schur diagonal of A^T A after i pivots, and R(i, j) = S(p, j) / sqrt(S(p, p)) up to
// the sign of row i (T = R11^-1 R12 and every |R| used by dlaqp2 are sign-invariant). So:
//
//   1. k_gid_count / k_gid_copy : gather A_{R,I} (m x k, column-major) with P CTAs per separator;
//   2. k_gid_gram               : G = A^T A, lower 64x64 tiles on DMMA (K = m streamed, cp.async);
//   3. k_gid_cpqr               : pivoted Cholesky of G on a thread-block cluster, replaying dlaqp2
//                                 exactly (pivot = first max of the partial norms vn1, swap
//                                 semantics, norm downdate with the tol3z recompute rule, where the
//                                 recomputed norm is the square root of the exact Schur diagonal),
//                                 the early stop of cta_cpqr, count-based rank; then
//                                 T = R11^-1 R12 by blocked back substitution across the cluster.
//
// The Schur complement is stored column-cyclic across the cluster's CTAs (full column b lives in
// CTA b % C), in shared memory up to the CTA's budget and the remaining columns in a global spill
// area. Partial norms, Schur diagonal and column positions are replicated in every CTA and
// updated with identical arithmetic, so every CTA selects the same pivot without communication;
// the only exchange per pivot step is row i of R (each CTA computes the entries of the columns
// it owns and pushes them to every CTA through distributed shared memory).

struct GidSmem {   // shared-memory carve-up (doubles first, then ints)
  // [Schur region sreg][panel nb x k][d, vn1, vn2: 3k][row pieces 2k][rdv, invv: 2k][96] doubles, then 3k ints
  // (the 96: argmax scratch, two mbarriers, and 2 x 16 step-token slots of the row exchange)
  __host__ __device__ static int64_t doubles(int64_t sreg, int k, int nb) {
    return sreg + (int64_t)(nb + 7) * k + 96;
  }
  __host__ __device__ static size_t bytes(int64_t sreg, int k, int nb) {
    return (size_t)doubles(sreg, k, nb) * sizeof(double) + 3 * (size_t)k * sizeof(int);
  }
};

// largest per-CTA share of the Schur complement (full owned columns)
__host__ __device__ __forceinline__ int64_t gid_pack0(int k, int C) { return (int64_t)((k + C - 1) / C) * k; }

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// generic address of the same shared-memory location in cluster CTA `rank` (plain loads through
// it stay ordinary memory operations, so the compiler keeps them behind the cluster barrier)
__device__ __forceinline__ const double* dsmem_map(const double* p, unsigned rank) {
  uint64_t out;
  asm("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"(reinterpret_cast<uint64_t>(p)), "r"(rank));
  return reinterpret_cast<const double*>(out);
}

// y[a] -= alpha * x[a] for a in [lo, hi), lanes of one warp; U loads in flight per lane before
// any store (x and y may alias as far as the compiler knows)
template <int U>
__device__ __forceinline__ void warp_axpy(double* y, const double* x, double alpha, int lo, int hi, int lane) {
  for (int a0 = lo + lane; a0 < hi; a0 += 32 * U) {
    double xv[U], yv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int a = a0 + 32 * u;
      xv[u] = a < hi ? x[a] : 0.0;
      yv[u] = a < hi ? y[a] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int a = a0 + 32 * u;
      if (a < hi) y[a] = __fma_rn(-xv[u], alpha, yv[u]);
    }
  }
}

// ---- 1. gather --------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) k_gid_count(LevelDev lv, SkelArgs sk, GramArgs ga) {
  __shared__ NbrCache nc;
  __shared__ int sbuf[1024];
  const int item = blockIdx.x / ga.P, part = blockIdx.x % ga.P;
  const int s = ga.item_sep[item];
  nbr_cache_load(lv, sk, s, nc);
  const int nch = nc.nch;
  const int lo = (int)((int64_t)nch * part / ga.P), hi = (int)((int64_t)nch * (part + 1) / ga.P);
  const int n = gather_chunks<false>(lv, sk, nc, s, lo, hi, nullptr, 1, 0, sbuf, 512);
  if (threadIdx.x == 0) ga.cnt[blockIdx.x] = n;
}

__global__ void __launch_bounds__(NT) k_gid_copy(LevelDev lv, SkelArgs sk, GramArgs ga) {
  __shared__ NbrCache nc;
  __shared__ int sbuf[1024];
  __shared__ int s_base, s_tot;
  const int item = blockIdx.x / ga.P, part = blockIdx.x % ga.P;
  const int s = ga.item_sep[item];
  if (threadIdx.x == 0) {
    int b = 0, t = 0;
    for (int q = 0; q < ga.P; ++q) {
      const int v = ga.cnt[item * ga.P + q];
      if (q < part) b += v;
      t += v;
    }
    s_base = b;
    s_tot = t;
  }
  nbr_cache_load(lv, sk, s, nc);   // (contains __syncthreads)
  const int nch = nc.nch;
  const int lo = (int)((int64_t)nch * part / ga.P), hi = (int)((int64_t)nch * (part + 1) / ga.P);
  double* W = sk.work + sk.work_off[s];
  gather_chunks<true, 16>(lv, sk, nc, s, lo, hi, W, ga.item_ld[item], s_base, sbuf, 512);
  if (part == 0 && threadIdx.x == 0) sk.rows[s] = s_tot;
}

// ---- 2. Gram tiles: G(a, b) = sum_r A(r, a) A(r, b), 64x64 lower tiles ----------------------
// Same pipeline as k_big_nt (K streamed in 32-wide chunks, 3 cp.async stages, DMMA m8n8k4):
// column a of A (contiguous over r) is the "row" a of the NT product. G is column-major (ld k).
__global__ void __launch_bounds__(NT, 2) k_gid_gram(LevelDev lv, SkelArgs sk, GramArgs ga) {
  extern __shared__ double smem[];
  const int item = ga.w_item[blockIdx.x], it = ga.w_i[blockIdx.x], jt = ga.w_j[blockIdx.x] & 0xffff;
  const int ks = ga.w_j[blockIdx.x] >> 16;   // split-K part: rows [kbeg, kend) into partial block ks
  const int s = ga.item_sep[item];
  const int k = lv.gsize[sk.groups[s]];
  const int mrows = sk.rows[s];
  const int kchunk = ((mrows + ga.S - 1) / ga.S + NTK - 1) / NTK * NTK;
  const int kbeg = min(mrows, ks * kchunk), m = min(mrows, kbeg + kchunk);
  const int64_t ld = ga.item_ld[item];
  const double* W = sk.work + sk.work_off[s];
  double* Gm = ga.gbuf + ga.g_off[item] + (int64_t)ks * k * k;
  const int ar0 = BT * it, br0 = BT * jt;
  const int Mv = min(BT, k - ar0), Nv = min(BT, k - br0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 3, wn = warp >> 2, g = lane >> 2, t = lane & 3;
  const double* Ab = W + (int64_t)ar0 * ld;
  const double* Bb = W + (int64_t)br0 * ld;
  auto load = [&](int st, int kc) {
    double* sA = smem + st * NT_STAGE;
    double* sB = sA + BT * NTLD;
#pragma unroll
    for (int q = 0; q < (BT * NTK) / NT; ++q) {
      const int e = tid + q * NT, r = e / NTK, kk = e % NTK;
      const int gk = kc + kk;
      const bool okA = r < Mv && gk < m, okB = r < Nv && gk < m;
      cp_async8(sA + r * NTLD + kk, Ab + (okA ? (int64_t)r * ld + gk : 0), okA);
      cp_async8(sB + r * NTLD + kk, Bb + (okB ? (int64_t)r * ld + gk : 0), okB);
    }
    cp_async_commit();
  };
  double acc[2][4][2];
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  const int nch = (m - kbeg + NTK - 1) / NTK;
  if (nch > 0) load(0, kbeg);
  if (nch > 1) load(1, kbeg + NTK);
  for (int ch = 0; ch < nch; ++ch) {
    if (ch + 2 < nch) {
      load((ch + 2) % NT_STAGES, kbeg + (ch + 2) * NTK);
      cp_async_wait<2>();
    } else if (ch + 1 < nch) {
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* sA = smem + (ch % NT_STAGES) * NT_STAGE;
    const double* sB = sA + BT * NTLD;
#pragma unroll
    for (int ks = 0; ks < NTK; ks += 4) {
      double af[2], bf[4];
#pragma unroll
      for (int x = 0; x < 2; ++x) af[x] = sA[(wm * 16 + x * 8 + g) * NTLD + ks + t];
#pragma unroll
      for (int y = 0; y < 4; ++y) bf[y] = sB[(wn * 32 + y * 8 + g) * NTLD + ks + t];
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) dmma(acc[x][y][0], acc[x][y][1], af[x], bf[y]);
    }
    __syncthreads();
  }
  // epilogue staged in the drained pipeline buffers, then coalesced column-major stores of the
  // tile and of its mirror (full G)
  double* sT = smem;
  constexpr int LD = BT + 1;
  if (nch == 0) __syncthreads();
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int z = 0; z < 2; ++z) {
        const int i = wm * 16 + x * 8 + g, j = wn * 32 + y * 8 + 2 * t + z;
        sT[j * LD + i] = acc[x][y][z];
      }
  __syncthreads();
  for (int e = tid; e < BT * BT; e += NT) {
    const int j = e / BT, i = e % BT;   // G(ar0 + i, br0 + j) at column br0 + j
    if (i < Mv && j < Nv) Gm[(int64_t)(br0 + j) * k + ar0 + i] = sT[j * LD + i];
  }
  if (it != jt)
    for (int e = tid; e < BT * BT; e += NT) {
      const int i = e / BT, j = e % BT;   // mirror G(br0 + j, ar0 + i) at column ar0 + i
      if (i < Mv && j < Nv) Gm[(int64_t)(ar0 + i) * k + br0 + j] = sT[j * LD + i];
    }
}

// ---- 3. pivoted Cholesky (dlaqp2 replay) + T on a cluster of C CTAs ------------------------
// CTA c owns the full columns b = c, c+C, ... of the Schur complement (shared memory up to its
// budget, the rest in a global spill area). Updates are deferred over panels of nb pivot steps
// (the panel's rows of R are replicated in shared memory): step i forms only row i,
// R(i, b) = (S(p, b) - sum_{l in panel} R(l, p) R(l, b)) / R(i, i), each CTA for its own columns,
// and pushes those entries into every CTA's row buffer with st.async, completing bytes on the
// receiver's mbarrier (no cluster-wide barrier per step). The owned columns receive the
// panel's rank-nb update once per panel.
constexpr int GID_NBMAX = 16;
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, unsigned rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const uint32_t a = smem_addr(bar);
  unsigned ok = 0;
  while (!ok)
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
}
__device__ __forceinline__ void st_async_f64(uint32_t raddr, double v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
               "l"(__double_as_longlong(v)), "r"(rbar)
               : "memory");
}

__global__ void __launch_bounds__(NT, 1) k_gid_cpqr(LevelDev lv, SkelArgs sk, GramArgs ga, int64_t sreg) {
  extern __shared__ double smem[];
  const int C = ga.C, nb = ga.nb;
  const int item = blockIdx.x / C;
  const int c = C > 1 ? (int)cluster_rank() : 0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = NT / 32;
  const int s = ga.item_sep[item];
  const int g = sk.groups[s], k = lv.gsize[g];
  const int64_t gof = lv.goff[g];
  const int m = sk.rows[s];
  if (m == 0) {   // uniform across the cluster: no coupling, every column redundant
    if (c == 0) skel_all_redundant(lv, sk, s);
    return;
  }
  const bool pf = ga.prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
  long long t0 = pf ? clock64() : 0;
#define GID_MARK(slot)                                                                                  \
  if (pf) {                                                                                             \
    const long long t1 = clock64();                                                                     \
    atomicAdd(reinterpret_cast<unsigned long long*>(ga.prof + (slot)), (unsigned long long)(t1 - t0)); \
    t0 = t1;                                                                                            \
  }
  const int nown0 = (k + C - 1) / C;
  double* Gm = ga.gbuf + ga.g_off[item];                              // G (full), then R (R(i, b) at Gm[b*k + i])
  const int64_t kk2 = (int64_t)k * k;
  double* Sg = Gm + ga.S * kk2 + (int64_t)c * nown0 * k;            // spill area (when allocated)
  double* Pn = smem + sreg;                 // nb x k panel rows of R
  double* d = Pn + (int64_t)nb * k;         // Schur diagonal (replicated)
  double* vn1 = d + k;
  double* vn2 = vn1 + k;
  double* rowbuf = vn2 + k;                 // 2 x k receive buffers (step parity)
  double* rdv = rowbuf + 2 * (int64_t)k;    // sqrt(Schur diagonal) and its reciprocal per column,
  double* invv = rdv + k;                   // formed off the pivot chain in the downdate loop
  double* sred = invv + k;                  // 96 (sred[48..49]: the two mbarriers, [64..95] tokens)
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sred + 48);
  double* tok = sred + 64;                  // tok[q * 16 + src]: step tokens (never read)
  int* col_at = reinterpret_cast<int*>(sred + 96);
  int* piv = col_at + k;
  int* sidx = piv + k;
  const int nown = c < k ? (k - c + C - 1) / C : 0;
  const int nsm = (int)(sreg / k < nown ? sreg / k : nown);   // owned columns resident in shared memory
  auto colf = [&](int lb) -> double* { return lb < nsm ? smem + (int64_t)lb * k : Sg + (int64_t)(lb - nsm) * k; };
  for (int lb = warp; lb < nown; lb += nw) {
    const int b = lb * C + c;
    double* col = colf(lb);
    const double* src = Gm + (int64_t)b * k;
    for (int a0 = lane; a0 < k; a0 += 32 * 4) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = a0 + 32 * u < k ? src[a0 + 32 * u] : 0.0;
      for (int q = 1; q < ga.S; ++q)   // split-K partial blocks, fixed order
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] += a0 + 32 * u < k ? src[q * kk2 + a0 + 32 * u] : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (a0 + 32 * u < k) col[a0 + 32 * u] = v[u];
    }
  }
  // vn1 / vn2 hold squared partial norms (argmax and the dlaqp2 tests in squared form)
  ArgMax loc{-1.0, 0x7fffffff};
  for (int j = tid; j < k; j += NT) {
    double dj = Gm[(int64_t)j * k + j];
    for (int q = 1; q < ga.S; ++q) dj += Gm[q * kk2 + (int64_t)j * k + j];
    const double nj = fmax(dj, 0.0);
    d[j] = dj;
    rdv[j] = sqrt(nj);
    invv[j] = nj > 0.0 ? 1.0 / rdv[j] : 0.0;
    vn1[j] = vn2[j] = nj;
    col_at[j] = j;
    piv[j] = 0;
    loc = better(loc, ArgMax{nj, j});
  }
  if (C > 1 && tid == 0) {
    mbar_init(mbar, 1);
    mbar_init(mbar + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  ArgMax best = cta_argmax1(loc, sred);
  if (C > 1) cluster_barrier();   // G read, mbarriers initialised cluster-wide
  else __syncthreads();
  GID_MARK(0)
  const uint32_t rb_addr = smem_addr(rowbuf), bar_addr = smem_addr(mbar), tok_addr = smem_addr(tok);
  // Back-pressure of the row exchange: besides its row entries, every CTA pushes one 8-byte token
  // per step to every CTA (also when none of its columns is still active), and every receiver
  // expects 8 (k - i - 1) + 8 C bytes. A CTA therefore completes step i + 1 only after every
  // peer has issued its step-(i + 1) pushes, i.e. after every peer has finished reading its own
  // step-i row buffer, so no CTA runs more than one step ahead: the step-(i + 2) pushes into
  // buffer parity q can never land while a peer still reads that buffer for step i.
  const uint32_t tok_dst = (C > 1 && tid < C) ? mapa_u32(tok_addr, (unsigned)tid) : 0u;
  const uint32_t tokbar_dst = (C > 1 && tid < C) ? mapa_u32(bar_addr, (unsigned)tid) : 0u;
  // threads per owned column in the row-entry step (power of two, nown <= NT / tpc when possible;
  // tpc >= C / 4 so every thread pushes to at most 4 destinations)
  int tpc = 8;
  while (tpc > 1 && nown > NT / tpc) tpc >>= 1;
  while (tpc * 4 < C) tpc <<= 1;
  // remote row-buffer / mbarrier addresses of the destinations this thread pushes to
  uint32_t rb_dst[4] = {0u, 0u, 0u, 0u}, bar_dst[4] = {0u, 0u, 0u, 0u};
  if (C > 1)
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int dst = (tid & (tpc - 1)) + tpc * u;
      if (dst < C) {
        rb_dst[u] = mapa_u32(rb_addr, (unsigned)dst);
        bar_dst[u] = mapa_u32(bar_addr, (unsigned)dst);
      }
    }
  const double tol3z = sqrt(DBL_EPSILON * 0.5);
  const double cutrel = fmax(sk.eps, DBL_EPSILON * (double)max(m, k));
  const int mn = min(m, k);
  double cut = 0.0, cut2 = 0.0;
  int r = 0, i = 0, np = 0;
  for (; i < mn; ++i) {
    if (i > 0 && best.v < cut2) break;
    const int q = i & 1;
    if (C > 1 && tid == 0) mbar_expect(mbar + q, 8u * (unsigned)(k - i - 1 + C));
    // pivot column (position best.i); the position swap is applied after the row exchange
    const int p = col_at[best.i];
    const double rd = i == 0 ? rdv[p] : sqrt(fmax(d[p], 0.0));   // (only the pivot needs it)
    if (i == 0) {
      cut = cutrel * rd;
      cut2 = cut * (1.0 - 1e-4) * (cut * (1.0 - 1e-4));
    }
    if (rd > cut) ++r;
    const double inv = i == 0 ? invv[p] : (rd > 0.0 ? 1.0 / rd : 0.0);
    double* row = Pn + (int64_t)np * k;   // this step's row of R
    // entries of row i in the owned columns, tpc threads per column (panel terms split tpc ways;
    // one round over the owned columns whenever nown <= 256)
    for (int cb0 = 0; cb0 < nown; cb0 += NT / tpc) {
      const int lb = cb0 + tid / tpc, part = tid & (tpc - 1);
      const int b = lb * C + c;
      const bool act = lb < nown && b != p && !piv[b];
      double v = 0.0;
      if (act) {
        for (int l = part; l < np; l += tpc) v = __fma_rn(-Pn[l * k + p], Pn[l * k + b], v);
        if (part == 0) v += colf(lb)[p];
      }
      for (int o = 1; o < tpc; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (act) {
        v *= inv;
        if (C > 1) {
          const uint32_t off = (uint32_t)(q * k + b) * 8u;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (part + u * tpc < C) st_async_f64(rb_dst[u] + off, v, bar_dst[u] + 8u * q);
        } else if (part == 0) {
          row[b] = v;
        }
      }
    }
    if (C > 1 && tid < C) st_async_f64(tok_dst + 8u * (uint32_t)(q * 16 + c), 0.0, tokbar_dst + 8u * q);
    GID_MARK(2)
    // C > 1: no CTA barrier here -- after the mbarrier wait every thread reads the received row
    // entries of its own downdate positions straight from the receive buffer and files them into
    // the panel row and (owned columns) into R; thread 0 files the diagonal. Entries of already
    // pivoted columns are never read again (row formation and downdates touch unpivoted columns
    // only; the back substitution reads R on and above the diagonal).
    const double* rb = rowbuf + (int64_t)q * k;
    if (C > 1) {
      mbar_wait(mbar + q, (unsigned)((i >> 1) & 1));
      GID_MARK(3)
      if (tid == 0) {
        row[p] = rd;
        piv[p] = 1;   // (read again only after the argmax barrier)
        if (p % C == c) Gm[(int64_t)p * k + i] = rd;
      }
    } else {
      __syncthreads();
      for (int a = tid; a < k; a += NT)
        if (a == p) row[a] = rd;
        else if (piv[a]) row[a] = 0.0;
      __syncthreads();
      if (tid == 0) piv[p] = 1;   // (read again only after the argmax barrier)
      for (int lb = tid; lb < nown; lb += NT) {   // row i of R, columns owned here
        const int b = lb * C + c;
        Gm[(int64_t)b * k + i] = row[b];
      }
    }
    GID_MARK(4)
    // fused: Schur diagonal, dlaqp2 partial-norm downdate and the next pivot's argmax over the
    // positions > i (identical arithmetic in every CTA)
    // the dlaqp2 swap of positions i and best.i is done by the thread owning position best.i
    // (it takes over position i's column and norms; position i is final)
    loc = ArgMax{-1.0, 0x7fffffff};
    const int pb = best.i;
    for (int j = i + 1 + tid; j < k; j += NT) {
      int col;
      if (j == pb) {
        col = col_at[i];
        col_at[j] = col;
        col_at[i] = p;
        vn1[j] = vn1[i];
        vn2[j] = vn2[i];
      } else {
        col = col_at[j];
      }
      double rv;
      if (C > 1) {
        rv = rb[col];
        row[col] = rv;
        if (col % C == c) Gm[(int64_t)col * k + i] = rv;
      } else {
        rv = row[col];
      }
      const double dn = __fma_rn(-rv, rv, d[col]);
      d[col] = dn;
      double w1 = vn1[j];
      if (w1 != 0.0) {
        // dlaqp2: temp = max(0, 1 - (|R(i,j)|/vn1)^2); recompute when temp (vn1/vn2)^2 <= tol3z,
        // else vn1 *= sqrt(temp) -- here on squared norms: w = vn1^2 - R(i,j)^2
        const double w = fmax(__fma_rn(-rv, rv, w1), 0.0);
        if (w <= tol3z * vn2[j]) {
          w1 = i < m - 1 ? fmax(dn, 0.0) : 0.0;
          vn2[j] = w1;
        } else {
          w1 = w;
        }
        vn1[j] = w1;
      }
      loc = better(loc, ArgMax{w1, j});
    }
    best = cta_argmax1(loc, sred);
    GID_MARK(6)
    if (++np == nb) {   // rank-nb update of the owned, unpivoted columns (all rows)
      // one warp per pair of owned columns, two rows per lane: each panel value loaded from shared
      // memory feeds two FMAs, four independent accumulation chains per lane
      for (int lp = warp; 2 * lp < nown; lp += nw) {
        const int lb1 = 2 * lp, lb2 = 2 * lp + 1;
        const bool u1 = !piv[lb1 * C + c], u2 = lb2 < nown && !piv[lb2 * C + c];
        if (!u1 && !u2) continue;
        double r1[GID_NBMAX], r2[GID_NBMAX];
#pragma unroll
        for (int l = 0; l < GID_NBMAX; ++l) {
          r1[l] = (u1 && l < np) ? Pn[l * k + lb1 * C + c] : 0.0;
          r2[l] = (u2 && l < np) ? Pn[l * k + lb2 * C + c] : 0.0;
        }
        double* c1 = colf(lb1);
        double* c2 = u2 ? colf(lb2) : c1;
        for (int a0 = lane; a0 < k; a0 += 64) {
          const int a1 = a0 + 32;
          const bool ok1 = a1 < k;
          double x00 = c1[a0], x01 = ok1 ? c1[a1] : 0.0, x10 = c2[a0], x11 = ok1 ? c2[a1] : 0.0;
#pragma unroll
          for (int l = 0; l < GID_NBMAX; ++l)
            if (l < np) {
              const double pa = Pn[l * k + a0], pb = ok1 ? Pn[l * k + a1] : 0.0;
              x00 = __fma_rn(-pa, r1[l], x00);
              x01 = __fma_rn(-pb, r1[l], x01);
              x10 = __fma_rn(-pa, r2[l], x10);
              x11 = __fma_rn(-pb, r2[l], x11);
            }
          if (u1) {
            c1[a0] = x00;
            if (ok1) c1[a1] = x01;
          }
          if (u2) {
            c2[a0] = x10;
            if (ok1) c2[a1] = x11;
          }
        }
      }
      np = 0;
      __syncthreads();
      GID_MARK(5)
    }
  }
  if (pf) atomicAdd(reinterpret_cast<unsigned long long*>(ga.prof + 9), (unsigned long long)i);
  const int kt = k - r;
  // redundant flags by column (positions r..k-1) and the sorted-list index of every column
  for (int j = tid; j < k; j += NT) piv[col_at[j]] = j >= r ? 1 : 0;
  __syncthreads();
  if (warp == 0) {
    int ns = 0, nr = 0;
    for (int j0 = 0; j0 < k; j0 += 32) {
      const int j = j0 + lane;
      const bool ok = j < k;
      const int f = ok ? piv[j] : 0;
      const unsigned bf = __ballot_sync(0xffffffffu, ok && f), bs = __ballot_sync(0xffffffffu, ok && !f);
      const unsigned below = (1u << lane) - 1u;
      if (ok) sidx[j] = f ? nr + __popc(bf & below) : ns + __popc(bs & below);
      nr += __popc(bf);
      ns += __popc(bs);
    }
  }
  __threadfence();
  if (C > 1) cluster_barrier();   // all rows of R in global memory; no more remote reads
  else __syncthreads();
  GID_MARK(7)
  // T = R11^-1 R12 (pivot order) by column back substitution; RHS columns spread over the
  // cluster's warps, 16/32-column blocks of R11 staged in shared memory (Schur region + panel)
  if (kt > 0 && r > 0) {
    double* T = sk.rec + sk.T_off[s];
    double* stage = smem;
    const int64_t sreg2 = sreg + (int64_t)nb * k;
    // staging: BW columns of R11 + NR right-hand sides per warp (host guarantees 24 k <= sreg2)
    const int BW = sreg2 >= (int64_t)(32 + nw) * r ? 32 : 16;
    const int NR = max(1, min(4, (int)((sreg2 / r - BW) / nw)));
    double* Rs = stage;
    double* xs = stage + (int64_t)BW * r + (int64_t)warp * NR * r;
    const int gw = c * nw + warp, nwarps = nw * C;
    const int ngroups = (kt + NR - 1) / NR;
    const int rounds = (ngroups + nwarps - 1) / nwarps;
    for (int round = 0; round < rounds; ++round) {
      const int q = round * nwarps + gw;
      const bool act = q < ngroups;
      const int j0 = q * NR, nj = act ? min(NR, kt - j0) : 0;
      for (int n = 0; n < nj; ++n) {
        const double* src = Gm + (int64_t)col_at[r + j0 + n] * k;
        for (int l = lane; l < r; l += 32) xs[n * r + l] = __ldcg(src + l);
      }
      __syncwarp();
      for (int i0 = ((r - 1) / BW) * BW; i0 >= 0; i0 -= BW) {
        const int ib = min(BW, r - i0), h = i0 + ib;
        __syncthreads();
        for (int e0 = tid; e0 < ib * h; e0 += 4 * NT) {
          double v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int e = e0 + u * NT;
            v[u] = e < ib * h ? __ldcg(Gm + (int64_t)col_at[i0 + e / h] * k + e % h) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int e = e0 + u * NT;
            if (e < ib * h) Rs[(e / h) * r + e % h] = v[u];
          }
        }
        __syncthreads();
        // all (up to 4) right-hand sides of the warp advance together: one staged R value feeds
        // nj FMAs, 4 rows per lane in flight
        for (int ii = ib - 1; ii >= 0 && nj > 0; --ii) {
          const int ia = i0 + ii;
          const double* Rc = Rs + ii * r;
          const double dinv = 1.0 / Rc[ia];
          double xi[4];
#pragma unroll
          for (int n = 0; n < 4; ++n) xi[n] = n < nj ? xs[n * r + ia] * dinv : 0.0;
          __syncwarp();
          if (lane == 0)
#pragma unroll
            for (int n = 0; n < 4; ++n)
              if (n < nj) xs[n * r + ia] = xi[n];
          for (int a0 = lane; a0 < ia; a0 += 128) {
            double rc[4], xv[4][4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int a = a0 + 32 * u;
              rc[u] = a < ia ? Rc[a] : 0.0;
#pragma unroll
              for (int n = 0; n < 4; ++n) xv[n][u] = (a < ia && n < nj) ? xs[n * r + a] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int a = a0 + 32 * u;
#pragma unroll
              for (int n = 0; n < 4; ++n)
                if (a < ia && n < nj) xs[n * r + a] = __fma_rn(-rc[u], xi[n], xv[n][u]);
            }
          }
          __syncwarp();
        }
      }
      for (int n = 0; n < nj; ++n) {
        const int cj = sidx[col_at[r + j0 + n]];
        for (int l = lane; l < r; l += 32) T[(int64_t)sidx[col_at[l]] * kt + cj] = xs[n * r + l];
      }
      __syncwarp();
    }
  }
  GID_MARK(8)
#undef GID_MARK
  if (c == 0) {
    uint8_t* redp = sk.red + gof;
    for (int j = tid; j < k; j += NT) {
      const int f = piv[j];
      redp[j] = (uint8_t)f;
      if (f) sk.alive[lv.mem[gof + j]] = 0;
    }
    if (tid == 0) sk.rank[s] = r;
  }
}
