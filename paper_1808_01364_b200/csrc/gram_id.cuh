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
// The Schur complement is stored packed-lower and column-cyclic across the cluster's CTAs
// (column b lives in CTA b % C, rows b..k-1), in shared memory up to the CTA's budget and the
// remaining columns in a global spill area. Partial norms, Schur diagonal and column positions are
// replicated in every CTA and updated with identical arithmetic, so every CTA selects the same
// pivot without communication; the only exchange per pivot step is row i of R (each CTA
// computes the entries of the columns it owns, one cluster barrier, then reads the row through
// distributed shared memory).

struct GidSmem {   // shared-memory carve-up (doubles first, then ints)
  // [Schur region sreg][panel nb x k][d, vn1, vn2: 3k][row pieces 2k][64] doubles, then 3k ints
  __host__ __device__ static int64_t doubles(int64_t sreg, int k, int nb) {
    return sreg + (int64_t)(nb + 5) * k + 64;
  }
  __host__ __device__ static size_t bytes(int64_t sreg, int k, int nb) {
    return (size_t)doubles(sreg, k, nb) * sizeof(double) + 3 * (size_t)k * sizeof(int);
  }
};

// packed-lower offset of CTA c's local column lb (global column b = lb*C + c, rows b..k-1)
__host__ __device__ __forceinline__ int64_t gid_coff(int lb, int k, int c, int C) {
  return (int64_t)lb * (k - c) - (int64_t)C * lb * (lb - 1) / 2;
}
__host__ __device__ __forceinline__ int64_t gid_pack0(int k, int C) {   // largest per-CTA packed size (c = 0)
  return gid_coff((k + C - 1) / C, k, 0, C);
}

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
  gather_chunks<true>(lv, sk, nc, s, lo, hi, W, ga.item_ld[item], s_base, sbuf, 512);
  if (part == 0 && threadIdx.x == 0) sk.rows[s] = s_tot;
}

// ---- 2. Gram tiles: G(a, b) = sum_r A(r, a) A(r, b), 64x64 lower tiles ----------------------
// Same pipeline as k_big_nt (K streamed in 32-wide chunks, 3 cp.async stages, DMMA m8n8k4):
// column a of A (contiguous over r) is the "row" a of the NT product. G is column-major (ld k).
__global__ void __launch_bounds__(NT, 2) k_gid_gram(LevelDev lv, SkelArgs sk, GramArgs ga) {
  extern __shared__ double smem[];
  const int item = ga.w_item[blockIdx.x], it = ga.w_i[blockIdx.x], jt = ga.w_j[blockIdx.x];
  const int s = ga.item_sep[item];
  const int k = lv.gsize[sk.groups[s]];
  const int m = sk.rows[s];
  const int64_t ld = ga.item_ld[item];
  const double* W = sk.work + sk.work_off[s];
  double* Gm = ga.gbuf + ga.g_off[item];
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
  const int nch = (m + NTK - 1) / NTK;
  if (nch > 0) load(0, 0);
  if (nch > 1) load(1, NTK);
  for (int ch = 0; ch < nch; ++ch) {
    if (ch + 2 < nch) {
      load((ch + 2) % NT_STAGES, (ch + 2) * NTK);
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
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int z = 0; z < 2; ++z) {
        const int i = wm * 16 + x * 8 + g, j = wn * 32 + y * 8 + 2 * t + z;
        if (i < Mv && j < Nv) Gm[(int64_t)(br0 + j) * k + ar0 + i] = acc[x][y][z];
      }
}

// ---- 3. pivoted Cholesky (dlaqp2 replay) + T on a cluster of C CTAs ------------------------
// Updates of the Schur complement are deferred over panels of nb pivot steps (the panel's rows
// of R are replicated in shared memory): a step only forms the entries of row i it needs,
// S(p, b) - sum_{l in panel} R(l, p) R(l, b), and the owned columns receive the panel's rank-nb
// update once per panel.
constexpr int GID_NBMAX = 16;
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
  double* Gm = ga.gbuf + ga.g_off[item];                              // G, then R (R(i, b) at Gm[b*k + i])
  double* Sg = Gm + (int64_t)k * k + (int64_t)c * gid_pack0(k, C);   // spill area (when allocated)
  double* Pn = smem + sreg;                 // nb x k panel rows of R
  double* d = Pn + (int64_t)nb * k;         // Schur diagonal (replicated)
  double* vn1 = d + k;
  double* vn2 = vn1 + k;
  double* rowbuf = vn2 + k;                 // 2 x k row pieces (step parity), read by the cluster
  double* sred = rowbuf + 2 * (int64_t)k;   // 64
  int* col_at = reinterpret_cast<int*>(sred + 64);
  int* piv = col_at + k;
  int* sidx = piv + k;
  const int nown = c < k ? (k - c + C - 1) / C : 0;
  // owned columns 0..nsm-1 in shared memory, the rest spilled to global memory
  int nsm = 0;
  while (nsm < nown && gid_coff(nsm + 1, k, c, C) <= sreg) ++nsm;
  const int64_t split = gid_coff(nsm, k, c, C);
  auto colp = [&](int lb) -> double* {   // S(., b) - b for owned column b = lb*C + c
    const int64_t o = gid_coff(lb, k, c, C);
    return (o < split ? smem + o : Sg + (o - split)) - (lb * C + c);
  };
  for (int lb = warp; lb < nown; lb += nw) {
    const int b = lb * C + c;
    double* col = colp(lb);
    const double* src = Gm + (int64_t)b * k;
    for (int a0 = b + lane; a0 < k; a0 += 32 * 4) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = a0 + 32 * u < k ? src[a0 + 32 * u] : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (a0 + 32 * u < k) col[a0 + 32 * u] = v[u];
    }
  }
  ArgMax loc{-1.0, 0x7fffffff};
  for (int j = tid; j < k; j += NT) {
    const double dj = Gm[(int64_t)j * k + j];
    const double nj = sqrt(fmax(dj, 0.0));
    d[j] = dj;
    vn1[j] = vn2[j] = nj;
    col_at[j] = j;
    piv[j] = 0;
    loc = better(loc, ArgMax{nj, j});
  }
  ArgMax best = cta_argmax(loc, sred);
  if (C > 1) cluster_barrier();   // G fully read before it is overwritten by R
  else __syncthreads();
  GID_MARK(0)
  const double tol3z = sqrt(DBL_EPSILON * 0.5);
  const double cutrel = fmax(sk.eps, DBL_EPSILON * (double)max(m, k));
  const int mn = min(m, k);
  double cut = 0.0;
  int r = 0, i = 0, np = 0;
  for (; i < mn; ++i) {
    if (i > 0 && best.v < cut * (1.0 - 1e-4)) break;
    if (tid == 0 && best.i != i) {
      const int pp = best.i, tcol = col_at[pp];
      col_at[pp] = col_at[i];
      col_at[i] = tcol;
      vn1[pp] = vn1[i];
      vn2[pp] = vn2[i];
    }
    __syncthreads();
    const int p = col_at[i];
    const double rd = sqrt(fmax(d[p], 0.0));
    if (i == 0) cut = cutrel * rd;
    if (rd > cut) ++r;
    const double inv = rd > 0.0 ? 1.0 / rd : 0.0;
    double* row = Pn + (int64_t)np * k;                       // this step's row of R
    double* buf = C > 1 ? rowbuf + (int64_t)(i & 1) * k : row;
    // entries of row i in the owned columns: (S(p, b) - sum_l R(l, p) R(l, b)) / R(i, i)
    for (int lb = tid; lb < nown; lb += NT) {
      const int b = lb * C + c;
      if (b < p && !piv[b]) {
        double v0 = colp(lb)[p], v1 = 0.0;
        int l = 0;
        for (; l + 1 < np; l += 2) {
          v0 = __fma_rn(-Pn[l * k + p], Pn[l * k + b], v0);
          v1 = __fma_rn(-Pn[(l + 1) * k + p], Pn[(l + 1) * k + b], v1);
        }
        if (l < np) v0 = __fma_rn(-Pn[l * k + p], Pn[l * k + b], v0);
        buf[b] = (v0 + v1) * inv;
      }
    }
    const unsigned owner = (unsigned)(p % C);
    if (owner == (unsigned)c) {
      const double* cp = colp(p / C);
      for (int a = p + 1 + tid; a < k; a += NT) {
        double v = 0.0;
        if (!piv[a]) {
          double v0 = cp[a], v1 = 0.0;
          int l = 0;
          for (; l + 1 < np; l += 2) {
            v0 = __fma_rn(-Pn[l * k + a], Pn[l * k + p], v0);
            v1 = __fma_rn(-Pn[(l + 1) * k + a], Pn[(l + 1) * k + p], v1);
          }
          if (l < np) v0 = __fma_rn(-Pn[l * k + a], Pn[l * k + p], v0);
          v = (v0 + v1) * inv;
        }
        buf[a] = v;
      }
    }
    GID_MARK(2)
    if (C > 1) {
      __syncthreads();
      if (tid == 0) piv[p] = 1;
      cluster_barrier();
      GID_MARK(3)
      for (int a0 = tid; a0 < k; a0 += 4 * NT) {   // 4 remote loads in flight per thread
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int a = a0 + u * NT;
          v[u] = 0.0;
          if (a < k && a != p && !piv[a]) v[u] = *dsmem_map(buf + a, a < p ? (unsigned)(a % C) : owner);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int a = a0 + u * NT;
          if (a < k) row[a] = a == p ? rd : v[u];
        }
      }
    } else {
      for (int a = tid; a < k; a += NT)   // pivoted columns (other than p) read as 0
        if (piv[a] && a != p) row[a] = 0.0;
      if (tid == 0) {
        row[p] = rd;
        piv[p] = 1;
      }
    }
    __syncthreads();
    GID_MARK(4)
    for (int lb = tid; lb < nown; lb += NT) {   // row i of R, columns owned here
      const int b = lb * C + c;
      Gm[(int64_t)b * k + i] = row[b];
    }
    // fused: Schur diagonal, dlaqp2 partial-norm downdate and the next pivot's argmax over the
    // positions > i (identical arithmetic in every CTA)
    loc = ArgMax{-1.0, 0x7fffffff};
    for (int j = i + 1 + tid; j < k; j += NT) {
      const int col = col_at[j];
      const double rv = row[col];
      const double dn = __fma_rn(-rv, rv, d[col]);
      d[col] = dn;
      double v1 = vn1[j];
      if (v1 != 0.0) {
        // dlaqp2: temp = max(0, 1 - (|R(i,j)|/vn1)^2); recompute when temp (vn1/vn2)^2 <= tol3z,
        // else vn1 *= sqrt(temp) -- in division-free form: w = vn1^2 - R(i,j)^2
        const double w = fmax(__fma_rn(-rv, rv, v1 * v1), 0.0);
        const double v2 = vn2[j];
        if (w <= tol3z * v2 * v2) {
          v1 = i < m - 1 ? sqrt(fmax(dn, 0.0)) : 0.0;
          vn2[j] = v1;
        } else {
          v1 = sqrt(w);
        }
        vn1[j] = v1;
      }
      loc = better(loc, ArgMax{v1, j});
    }
    best = cta_argmax(loc, sred);
    GID_MARK(6)
    if (++np == nb) {   // rank-nb update of the owned, unpivoted columns
      for (int lb = warp; lb < nown; lb += nw) {
        const int b = lb * C + c;
        if (piv[b]) continue;
        double rb[GID_NBMAX];
#pragma unroll
        for (int l = 0; l < GID_NBMAX; ++l) rb[l] = l < np ? Pn[l * k + b] : 0.0;
        double* col = colp(lb);
        for (int a0 = b + 1 + lane; a0 < k; a0 += 64) {
          const int a1 = a0 + 32;
          double v0 = col[a0], v1 = a1 < k ? col[a1] : 0.0;
#pragma unroll
          for (int l = 0; l < GID_NBMAX; ++l)
            if (l < np) {
              v0 = __fma_rn(-Pn[l * k + a0], rb[l], v0);
              if (a1 < k) v1 = __fma_rn(-Pn[l * k + a1], rb[l], v1);
            }
          col[a0] = v0;
          if (a1 < k) col[a1] = v1;
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
        for (int ii = ib - 1; ii >= 0 && nj > 0; --ii) {
          const int ia = i0 + ii;
          const double* Rc = Rs + ii * r;
          const double dg = Rc[ia];
          for (int n = 0; n < nj; ++n) {
            double* x = xs + n * r;
            const double xi = x[ia] / dg;
            __syncwarp();
            if (lane == 0) x[ia] = xi;
            warp_axpy<4>(x, Rc, xi, 0, ia, lane);
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
