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
// area. Partial norms, Schur diagonal and position of a column live only in its owner; per pivot
// step the CTAs exchange one small candidate message each (see k_gid_cpqr) and every CTA forms
// only its own entries of row i of R.

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
// budget, the rest in a global spill area); rows are stored in the permuted order
// a' = (a % C) * nown0 + a / C, so every CTA's entries of a row of R are one contiguous segment.
//
// Candidate exchange. Norms, Schur diagonal and positions of a column live only in its owner
// (registers of warp 0, which runs the whole pivot chain without CTA barriers). Per step every
// CTA picks its local candidate (largest partial norm, lowest position among ties) and pushes one
// small message to every CTA of the cluster: [norm^2, (position, column), Schur diagonal, -, and the
// candidate column's entries in the current panel rows] (one word per lane, one st.async per
// lane and destination). After ONE mbarrier wait every CTA reduces
// the C candidates with the same rule -- the dlaqp2 pivot -- and already holds what it needs to
// form its own entries of row i,
//   R(i, b) = (S(p, b) - sum_{l in panel} R(l, p) R(l, b)) / R(i, i),   S(p, b) = S(b, p)' own column,
// and to downdate its own norms. Full rows of R are not exchanged on the pivot chain: the panel's
// rows are all-gathered once per panel (one bulk shared::cta -> shared::cluster copy per row and
// peer) right before the rank-nb update of the owned columns, which runs on DMMA with all warps.
// Flow control: a CTA completes step i only after every peer pushed its step-i message, which a
// peer does only after it finished reading the step-(i-1) slots and (at panel boundaries) its
// panel update; so the double-buffered slots and the single panel buffer are never overwritten
// while still in use.
constexpr int GID_NBMAX = 16;
struct GidShape {   // shapes shared by host and device
  int nown0, kp, lds, ldp;
  __host__ __device__ GidShape(int k, int C) {
    nown0 = ((k + C - 1) / C + 1) & ~1;   // owned columns per CTA, even (16-byte row segments)
    kp = (C * nown0 + 15) & ~15;          // permuted rows, padded for the 16-row DMMA blocks
    lds = kp + 2;                         // column stride of the Schur storage (= 2 mod 8) and
    ldp = kp + 4;                         // row stride of the panel (= 4 mod 16): conflict-free fragments
  }
};
struct GidSmem {   // shared-memory carve-up (doubles first, then ints)
  // [Schur region sreg][panel nb x ldp][candidate slots 2 x C x (nb + 4)][8: mbarriers, flags] doubles, then 3k ints
  __host__ __device__ static int64_t doubles(int64_t sreg, int k, int C, int nb) {
    return sreg + (int64_t)nb * GidShape(k, C).ldp + 2 * (int64_t)C * (nb + 4) + 8;
  }
  __host__ __device__ static size_t bytes(int64_t sreg, int k, int C, int nb) {
    return (size_t)doubles(sreg, k, C, nb) * sizeof(double) + 3 * (size_t)k * sizeof(int);
  }
};
// per-CTA share of the Schur complement (owned columns at their padded stride)
__host__ __device__ __forceinline__ int64_t gid_pack0(int k, int C) {
  const GidShape sh(k, C);
  return (int64_t)sh.nown0 * sh.lds;
}

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
__device__ __forceinline__ void st_async_b64(uint32_t raddr, unsigned long long v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr), "l"(v),
               "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void bulk_cta_to_cluster(uint32_t rdst, uint32_t src, uint32_t bytes, uint32_t rbar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(rdst),
               "r"(src), "r"(bytes), "r"(rbar)
               : "memory");
}
// UMAX: column slots per lane of the pivot-chain warp (owned columns per CTA <= 32 * UMAX)
template <int UMAX>
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
  const GidShape sh(k, C);
  const int nown0 = sh.nown0, kp = sh.kp, lds = sh.lds, ldp = sh.ldp;
  const int SLOT = nb + 4;
  double* Gm = ga.gbuf + ga.g_off[item];                              // G (full), then R (R(i, b) at Gm[b*k + i])
  const int64_t kk2 = (int64_t)k * k;
  double* Sg = Gm + ga.S * kk2 + (int64_t)c * nown0 * lds;          // spill area (when allocated)
  double* Pn = smem + sreg;                              // nb panel rows of R (permuted column order)
  double* slots = Pn + (int64_t)nb * ldp;                // [2][C][SLOT] candidate messages
  double* misc = slots + 2 * (int64_t)C * SLOT;          // 8: three mbarriers, flags
  uint64_t* mbar = reinterpret_cast<uint64_t*>(misc);    // [0], [1]: candidates (step parity), [2]: panel
  int* sflag = reinterpret_cast<int*>(misc + 3);         // [0] another panel follows, [1] rank, [2] steps
  int* col_at = reinterpret_cast<int*>(misc + 8);
  int* piv = col_at + k;
  int* sidx = piv + k;
  const int nown = c < k ? (k - c + C - 1) / C : 0;      // owned columns b = lb * C + c
  int nsm = (int)(sreg / lds < nown0 ? sreg / lds : nown0);   // owned columns resident in shared memory
  if (nsm < nown0) nsm &= ~7;                            // (whole 8-column DMMA tiles on either side)
  auto colf = [&](int lb) -> double* { return lb < nsm ? smem + (int64_t)lb * lds : Sg + (int64_t)(lb - nsm) * lds; };
  // own columns of G (split-K partial blocks summed in a fixed order), rows permuted, pads zero
  for (int lb = warp; lb < nown; lb += nw) {
    const int b = lb * C + c;
    double* col = colf(lb);
    const double* src = Gm + (int64_t)b * k;
    for (int a0 = lane; a0 < lds; a0 += 32 * 4) {
      double v[4];
      int a[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int ap = a0 + 32 * u;
        a[u] = (ap % nown0) * C + ap / nown0;
        if (ap >= C * nown0 || a[u] >= k) a[u] = -1;
        v[u] = a[u] >= 0 ? src[a[u]] : 0.0;
      }
      for (int q = 1; q < ga.S; ++q)
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] += a[u] >= 0 ? src[q * kk2 + a[u]] : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (a0 + 32 * u < lds) col[a0 + 32 * u] = v[u];
    }
  }
  for (int e = tid; e < nb * ldp; e += NT) Pn[e] = 0.0;
  for (int j = tid; j < k; j += NT) {
    col_at[j] = j;
    piv[j] = 0;
  }
  if (tid == 0) {
    mbar_init(mbar, 1);
    mbar_init(mbar + 1, 1);
    mbar_init(mbar + 2, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (C > 1) cluster_barrier();   // mbarriers initialised cluster-wide
  GID_MARK(0)
  const double* Pown = Pn + c * nown0;
  int npanel = 0;
  // all-gather of the panel's rows + rank-nb update of the owned columns (all threads)
  auto panel_end = [&]() {
    if (C > 1) {
      if (tid == 0) mbar_expect(mbar + 2, 8u * (unsigned)((C - 1) * nb * nown0));
      const uint32_t bar2 = smem_addr(mbar + 2);
      for (int e = tid; e < nb * (C - 1); e += NT) {
        const int l = e / (C - 1), dd = e % (C - 1), dst = dd + (dd >= c ? 1 : 0);
        const uint32_t src = smem_addr(Pown + l * ldp);
        bulk_cta_to_cluster(mapa_u32(src, (unsigned)dst), src, 8u * (unsigned)nown0, mapa_u32(bar2, (unsigned)dst));
      }
      mbar_wait(mbar + 2, (unsigned)(npanel & 1));
    }
    ++npanel;
    // S(a', lb) -= sum_l P(l, a') P(l, lb): 16-row blocks over the warps, 4 column tiles at a time
    const int g8 = lane >> 2, t4 = lane & 3;
    const int nct = (nown + 7) >> 3;
    for (int rb = warp; rb < (kp >> 4); rb += nw) {
      const int r0 = rb << 4;
      for (int ct0 = 0; ct0 < nct; ct0 += 4) {
        double acc[2][4][2];
        double* cp[4][2];
#pragma unroll
        for (int y = 0; y < 4; ++y)
#pragma unroll
          for (int z = 0; z < 2; ++z) {
            const int lb = (ct0 + y) * 8 + 2 * t4 + z;
            cp[y][z] = lb < nown ? colf(lb) + r0 + g8 : nullptr;
#pragma unroll
            for (int x = 0; x < 2; ++x) acc[x][y][z] = cp[y][z] ? cp[y][z][8 * x] : 0.0;
          }
        for (int ks = 0; ks < nb; ks += 4) {
          const double* pr = Pn + (ks + t4) * ldp;
          double af[2], bf[4];
#pragma unroll
          for (int x = 0; x < 2; ++x) af[x] = -pr[r0 + 8 * x + g8];
#pragma unroll
          for (int y = 0; y < 4; ++y) bf[y] = pr[c * nown0 + (ct0 + y) * 8 + g8];
#pragma unroll
          for (int x = 0; x < 2; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) dmma(acc[x][y][0], acc[x][y][1], af[x], bf[y]);
        }
#pragma unroll
        for (int y = 0; y < 4; ++y)
#pragma unroll
          for (int z = 0; z < 2; ++z)
            if (cp[y][z]) {
#pragma unroll
              for (int x = 0; x < 2; ++x) cp[y][z][8 * x] = acc[x][y][z];
            }
      }
    }
    __syncthreads();
  };
  if (warp != 0) {
    for (;;) {   // helpers: wait for a full panel (or the end of the pivot chain)
      __syncthreads();
      if (!sflag[0]) break;
      panel_end();
    }
  } else {
    // ---- the pivot chain (warp 0): own columns lb = lane + 32 u ----
    int cb[UMAX], cpos[UMAX];
    bool cpv[UMAX];            // pivoted (or no such column)
    double cd[UMAX], c1[UMAX], c2[UMAX];
#pragma unroll
    for (int u = 0; u < UMAX; ++u) {
      const int lb = lane + 32 * u;
      const bool ok = lb < nown;
      cb[u] = ok ? lb * C + c : -1;
      cpos[u] = cb[u];
      cpv[u] = !ok;
      const double dj = ok ? colf(lb)[c * nown0 + lb] : 0.0;
      cd[u] = dj;
      c1[u] = c2[u] = fmax(dj, 0.0);   // squared partial norms (argmax and the dlaqp2 tests in squared form)
    }
    const uint32_t slot_addr = smem_addr(slots), bar_addr = smem_addr(mbar);
    const double tol3z = sqrt(DBL_EPSILON * 0.5);
    const double cutrel = fmax(sk.eps, DBL_EPSILON * (double)max(m, k));
    const int mn = min(m, k);
    double cut = 0.0, cut2 = 0.0;
    const int lgC = 31 - __clz(C);
    int r = 0, i = 0, np = 0;
    for (; i < mn; ++i) {
      const int q = i & 1;
      // local candidate: largest partial norm, lowest position among ties
      double bv = 0.0, bd = 0.0;
      int bpos = 0x7fffffff, bcol = -1, blb = 0;
#pragma unroll
      for (int u = 0; u < UMAX; ++u)
        if (!cpv[u] && (c1[u] > bv || (c1[u] == bv && cpos[u] < bpos))) {
          bv = c1[u];
          bd = cd[u];
          bpos = cpos[u];
          bcol = cb[u];
          blb = lane + 32 * u;
        }
      const unsigned wm = warp_first_max(bv, (unsigned)bpos);
      const int wl = __ffs(wm) - 1;   // (bpos values are distinct except the "none" marker)
      const double wv = __shfl_sync(0xffffffffu, bv, wl);
      const int wpos = __shfl_sync(0xffffffffu, bpos, wl);
      const int wcol = __shfl_sync(0xffffffffu, bcol, wl);
      const int wlb = __shfl_sync(0xffffffffu, blb, wl);
      const double wd = __shfl_sync(0xffffffffu, bd, wl);
      // message word `word` of this lane: [norm^2, (position, column), Schur diagonal, panel entries]
      const int nwords = np + 4;   // (word 3 unused: the panel entries start 16-byte aligned)
      const int P2 = nwords <= 8 ? 8 : (nwords <= 16 ? 16 : 32);
      const int word = lane & (P2 - 1);
      unsigned long long val = 0ull;
      if (word == 0) val = (unsigned long long)__double_as_longlong(wv);
      else if (word == 1) val = ((unsigned long long)(unsigned)wpos << 32) | (unsigned)wcol;
      else if (word == 2) val = (unsigned long long)__double_as_longlong(wd);
      else if (word > 3 && word < nwords) val = (unsigned long long)__double_as_longlong(Pown[(word - 4) * ldp + wlb]);
      if (C > 1) {
        if (lane == 0) mbar_expect(mbar + q, 8u * (unsigned)(C * nwords));
        if (word < nwords) {
          // every lane sends its one word to the destinations d = lane / P2, + 32 / P2, ...
          const uint32_t off = (uint32_t)((q * C + c) * SLOT + word) * 8u;
          for (int dd = lane / P2; dd < C; dd += 32 / P2)
            st_async_b64(mapa_u32(slot_addr, (unsigned)dd) + off, val, mapa_u32(bar_addr, (unsigned)dd) + 8u * q);
        }
        GID_MARK(2)
        mbar_wait(mbar + q, (unsigned)((i >> 1) & 1));
        GID_MARK(3)
      } else {
        unsigned long long* ms = reinterpret_cast<unsigned long long*>(slots + (int64_t)(q * C + c) * SLOT);
        if (lane < nwords) ms[lane] = val;
        __syncwarp();
        GID_MARK(2)
      }
      // the pivot: first maximum over the C candidates (identical in every CTA)
      int ws = 0;
      if (C > 1) {
        double sv = 0.0;
        unsigned spos = 0xffffffffu;
        if (lane < C) {
          const double* sl = slots + (int64_t)(q * C + lane) * SLOT;
          sv = sl[0];
          spos = (unsigned)(reinterpret_cast<const unsigned long long*>(sl)[1] >> 32);
        }
        ws = __ffs(warp_first_max(sv, spos)) - 1;
      }
      const double* wsl = slots + (int64_t)(q * C + ws) * SLOT;
      const double gv = wsl[0];
      const unsigned long long key = reinterpret_cast<const unsigned long long*>(wsl)[1];
      const int pb = (int)(key >> 32), p = (int)(unsigned)key;
      // R_ii and 1 / R_ii of the pivot, formed by every CTA (they overlap the row's FMA chains)
      const double rd = sqrt(fmax(wsl[2], 0.0));
      const double inv = rd > 0.0 ? 1.0 / rd : 0.0;
      if (pb == 0x7fffffff) break;            // (no unpivoted column left: cannot happen while i < k)
      if (i > 0 && gv < cut2) break;
      if (i == 0) {
        cut = cutrel * rd;
        cut2 = cut * (1.0 - 1e-4) * (cut * (1.0 - 1e-4));
      }
      if (rd > cut) ++r;
      // own entries of row i of R
      const int pp = (p & (C - 1)) * nown0 + (p >> lgC);   // (C is a power of two)
      double* prow = Pn + np * ldp + c * nown0;
      double rp[GID_NBMAX];
#pragma unroll
      for (int l = 0; l < GID_NBMAX; l += 2) {   // (entries beyond np are stale and never used)
        double2 t2 = make_double2(0.0, 0.0);
        if (l < nb) t2 = *reinterpret_cast<const double2*>(wsl + 4 + l);
        rp[l] = t2.x;
        rp[l + 1] = t2.y;
      }
      double rvv[UMAX];
#pragma unroll
      for (int u = 0; u < UMAX; ++u) {
        const int lb = lane + 32 * u;
        rvv[u] = 0.0;
        if (cb[u] >= 0) {
          double v;
          if (cb[u] == p) {
            v = rd;
            cpv[u] = true;
            Gm[(int64_t)p * k + i] = rd;
          } else if (cpv[u]) {
            v = 0.0;
          } else {
            double acc = colf(lb)[pp];
#pragma unroll
            for (int l = 0; l < GID_NBMAX; ++l)
              if (l < np) acc = __fma_rn(-rp[l], Pown[l * ldp + lb], acc);
            v = acc * inv;
            Gm[(int64_t)cb[u] * k + i] = v;
            rvv[u] = v;
          }
          prow[lb] = v;
        }
      }
      // dlaqp2 swap of positions i and pb: the column displaced from position i moves to pb
      const int ci = col_at[i];
      __syncwarp();
      if (lane == 0) {
        col_at[pb] = ci;
        col_at[i] = p;
      }
      GID_MARK(4)
      // Schur diagonal and dlaqp2 partial-norm downdate of the own unpivoted columns
#pragma unroll
      for (int u = 0; u < UMAX; ++u)
        if (!cpv[u]) {
          if (cb[u] == ci) cpos[u] = pb;
          const double rv = rvv[u];
          const double dn = __fma_rn(-rv, rv, cd[u]);
          cd[u] = dn;
          double w1 = c1[u];
          if (w1 != 0.0) {
            // dlaqp2: temp = max(0, 1 - (|R(i,j)|/vn1)^2); recompute when temp (vn1/vn2)^2 <= tol3z,
            // else vn1 *= sqrt(temp) -- here on squared norms: w = vn1^2 - R(i,j)^2
            const double w = fmax(__fma_rn(-rv, rv, w1), 0.0);
            if (w <= tol3z * c2[u]) {
              w1 = i < m - 1 ? fmax(dn, 0.0) : 0.0;
              c2[u] = w1;
            } else {
              w1 = w;
            }
            c1[u] = w1;
          }
        }
      GID_MARK(6)
      if (++np == nb) {   // rank-nb update of the owned columns
        if (lane == 0) sflag[0] = 1;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // panel rows -> bulk copies
        __syncthreads();
        panel_end();
        np = 0;
        GID_MARK(5)
      }
    }
    if (lane == 0) {
      sflag[0] = 0;
      sflag[1] = r;
      sflag[2] = i;
    }
    __syncthreads();
  }
  const int r = sflag[1], i = sflag[2];
  if (pf) atomicAdd(reinterpret_cast<unsigned long long*>(ga.prof + 9), (unsigned long long)i);
  // redundant flags by column (positions r..k-1), the rank and the pivot order go out; T is formed
  // for all waves at once by k_gid_T after the last wave
  if (c == 0) {
    uint8_t* redp = sk.red + gof;
    int* colg = ga.col + ga.c_off[item];
    for (int j = tid; j < k; j += NT) {
      const int cj = col_at[j];
      const int f = j >= r ? 1 : 0;
      colg[j] = cj;
      redp[cj] = (uint8_t)f;
      if (f) sk.alive[lv.mem[gof + cj]] = 0;
    }
    if (tid == 0) sk.rank[s] = r;
  }
  __threadfence();
  if (C > 1) cluster_barrier();   // no CTA leaves while a peer's bulk copy may still read its panel
  GID_MARK(7)
#undef GID_MARK
}

// ---- 4. T = R11^-1 R12 of every Gram-path separator of the level (after the last wave) -------
// R(i, b) sits at Gm[b*k + i] (written by k_gid_cpqr), the pivot order in ga.col. CT CTAs per
// item; RHS columns spread over their warps, 16/32-column blocks of R11 staged in shared memory.
__global__ void __launch_bounds__(NT, 1) k_gid_T(LevelDev lv, SkelArgs sk, GramArgs ga) {
  extern __shared__ double smem[];
  const int C = ga.CT;
  const int item = blockIdx.x / C, c = blockIdx.x % C;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = NT / 32;
  const int s = ga.item_sep[item];
  const int g = sk.groups[s], k = lv.gsize[g];
  const int64_t gof = lv.goff[g];
  const int r = sk.rank[s], kt = k - r;
  if (kt == 0 || r == 0 || sk.rows[s] == 0) return;
  double* Gm = ga.gbuf + ga.g_off[item];
  int* col_at = reinterpret_cast<int*>(smem + ga.tcap);
  int* sidx = col_at + k;
  const uint8_t* redp = sk.red + gof;
  const int* colg = ga.col + ga.c_off[item];
  for (int j = tid; j < k; j += NT) col_at[j] = colg[j];
  if (warp == 0) {   // sorted-list index of every column inside its (skeleton / redundant) set
    int ns = 0, nr = 0;
    for (int j0 = 0; j0 < k; j0 += 32) {
      const int j = j0 + lane;
      const bool ok = j < k;
      const int f = ok ? redp[j] : 0;
      const unsigned bf = __ballot_sync(0xffffffffu, ok && f), bs = __ballot_sync(0xffffffffu, ok && !f);
      const unsigned below = (1u << lane) - 1u;
      if (ok) sidx[j] = f ? nr + __popc(bf & below) : ns + __popc(bs & below);
      nr += __popc(bf);
      ns += __popc(bs);
    }
  }
  __syncthreads();
  {
    double* T = sk.rec + sk.T_off[s];
    double* stage = smem;
    const int64_t sreg2 = ga.tcap;
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
}
