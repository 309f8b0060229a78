// Batched stage kernels of the B200 PHIF engine (sm_100a, FP64).
//
// One CTA per cell / group / block; all dense algebra through dla.cuh
// (DMMA GEMM core). Reference semantics are cited per kernel.
#include <algorithm>
#include <atomic>
#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

#include "dla.cuh"
#include "kernels.cuh"
#include "launch.h"

namespace phif {

static_assert(NT == 256, "kernels assume 256-thread CTAs");

__device__ __forceinline__ int find_blk(const int64_t* adj_off, const int* adj_nbr, const int* adj_blk, int g,
                                        int h) {
  int64_t lo = adj_off[g], hi = adj_off[g + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const int v = adj_nbr[mid];
    if (v < h) lo = mid + 1;
    else hi = mid;
  }
  if (lo < adj_off[g + 1] && adj_nbr[lo] == h) return adj_blk[lo];
  return -1;
}

__device__ __forceinline__ void report_bad(DevStatus* st, int op, int pivot) {
  const unsigned long long v = ((unsigned long long)(unsigned)op << 32) | (unsigned)pivot;
  atomicMin(&st->first_bad, v);
}

// ---------------------------------------------------------------------------
// Level-0 ingest: scatter the CSR of A into the dense group-pair blocks.
// ---------------------------------------------------------------------------
__global__ void k_ingest(LevelDev lv, const int* gid, const int* pos, const int64_t* rowptr, const int* col,
                         const double* val, int64_t N) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= N) return;
  const int g = gid[r], pr = pos[r];
  for (int64_t e = rowptr[r]; e < rowptr[r + 1]; ++e) {
    const int c = col[e];
    const int h = gid[c];
    if (h < g) continue;
    const int blk = find_blk(lv.adj_off, lv.adj_nbr, lv.adj_blk, g, h);
    if (blk < 0) continue;
    lv.pool[lv.boff[blk] + (int64_t)pr * lv.gsize[h] + pos[c]] = val[e];
  }
}

// group and position of every member DOF (one warp per group)
__global__ void k_group_pos(LevelDev lv, int* gid, int* pos) {
  const int w = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (w >= lv.G) return;
  const int64_t q0 = lv.goff[w], q1 = lv.goff[w + 1];
  for (int64_t q = q0 + lane; q < q1; q += 32) {
    const int d = lv.mem[q];
    gid[d] = w;
    pos[d] = (int)(q - q0);
  }
}

// ---------------------------------------------------------------------------
// Stage 1: cell elimination.
// Panel P = [A_II ; A_BI] ((n+b) x n) -> partial Cholesky -> [L ; X^T]; U = X^T X.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(NT, 3) k_cell(LevelDev lv, CellArgs ca, DevStatus* st) {
  extern __shared__ double smem[];
  const int t = ca.list ? ca.list[blockIdx.x] : blockIdx.x, tid = threadIdx.x;
  const int I = ca.interior[t], n = ca.n[t], b = ca.b[t];
  double* P = ca.rec + ca.P_off[t];
  const double* A = lv.pool + lv.boff[lv.diag_blk[I]];
  for (int64_t e = tid; e < (int64_t)n * n; e += NT) P[e] = A[e];
  for (int64_t j = ca.nbr_off[t]; j < ca.nbr_off[t + 1]; ++j) {
    const int w = ca.nbr_w[j], c0 = ca.nbr_col[j];
    const double* S = lv.pool + lv.boff[ca.nbr_blk[j]];
    for (int64_t e = tid; e < (int64_t)n * w; e += NT) {
      const int i = (int)(e / w), r = (int)(e % w);
      P[(int64_t)(n + c0 + r) * n + i] = S[e];
    }
  }
  double* Id = P + (int64_t)(n + b) * n;   // identity rows: become L^-T (GEMM replay)
  for (int64_t e = tid; e < (int64_t)n * n; e += NT) Id[e] = (e / n == e % n) ? 1.0 : 0.0;
  __syncthreads();
  const int info = cta_potrf_panel(P, n + b + n, n, n, smem);
  if (info >= 0) {
    if (tid == 0) report_bad(st, t, info);
    return;
  }
  if (b > 0)
    cta_gemm<false, true>(b, b, n, 1.0, P + (int64_t)n * n, n, P + (int64_t)n * n, n, 0.0, ca.U + ca.U_off[t], b,
                          false, smem + GEMM_OFF);
}

// ---------------------------------------------------------------------------
// Banded cells (2D level 0, n = (m-1)^2 interior DOFs in natural order): A_II is the 5-point
// stencil restricted to the cell, banded with half-bandwidth w = m-1 (checked on the device by
// k_band_check before this path is taken), so its Cholesky factor has the same band
// (POTRF n w^2, TRSM 2 n w b). One CTA per cell:
//   1. band of A_II -> shared memory; banded Cholesky by one warp (right-looking, no CTA
//      barriers on the column chain); NotSpd reported like the dense path (cell, 0-based pivot);
//   2. X = L^-1 A_BI^T: one thread per boundary DOF, forward substitution with the last w
//      values in registers, written straight into the panel rows [n, n+b) as X^T;
//   3. U = X^T X from 64-column chunks of X^T staged in shared memory;
//   4. the record rows: L (dense rows, zeros outside the band) and L^-T (row j = L^-1 e_j, one
//      thread per column of the identity), the layout the big-cell replay reads.
// ---------------------------------------------------------------------------
constexpr int BAND_WMAX = 31;   // w <= 31: one lane per band entry of a column
// Banded Cholesky of the level-0 cells, one warp per cell (many cells in flight per SM hide the
// per-column dependency chain): register window of w+1 rows, band of L and 1/diag to a scratch
// area read by k_cell_band; NotSpd reported like the dense path (cell, 0-based pivot).
template <int WM>
__global__ void __launch_bounds__(256) k_band_chol(LevelDev lv, CellArgs ca, const int* list, int count, int w,
                                                   double* scratch, int64_t stride, DevStatus* st) {
  const int wid = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (wid >= count) return;
  const int t = list[wid], I = ca.interior[t], n = ca.n[t];
  const int W1 = w + 1;
  const double* A = lv.pool + lv.boff[lv.diag_blk[I]];
  double* Lb = scratch + (int64_t)wid * stride;   // n x (w+1) band, then n reciprocals
  double* dinv = Lb + (int64_t)n * W1;
  // lane d <= w holds row j+d of the active band, R[c] = A(j+d, j+c) (c <= d); per column:
  // broadcast the pivot, scale the column, rank-1 update of the window (shuffles), shift the
  // window one row/column down and bring the next row in
  double R[WM + 1], nxt[WM + 1];
#pragma unroll
  for (int c = 0; c <= WM; ++c) R[c] = (lane <= w && c <= lane && lane < n) ? A[(int64_t)lane * n + c] : 0.0;
#pragma unroll
  for (int c = 0; c <= WM; ++c)   // the row entering after column 0 (loaded one column ahead)
    nxt[c] = (lane == w && 1 + w < n && c <= w) ? A[(int64_t)(1 + w) * n + 1 + c] : 0.0;
  for (int j = 0; j < n; ++j) {
    const double djj = __shfl_sync(0xffffffffu, R[0], 0);
    if (!(djj > 0.0)) {
      if (lane == 0) report_bad(st, t, j);
      return;
    }
    const double ljj = sqrt(djj), rinv = 1.0 / ljj;
    const bool row_ok = lane >= 1 && lane <= w && j + lane < n;
    const double cd = row_ok ? R[0] * rinv : 0.0;   // L(j+lane, j)
    if (lane == 0) {
      Lb[(int64_t)j * W1] = ljj;
      dinv[j] = rinv;
    } else if (row_ok) {
      Lb[(int64_t)(j + lane) * W1 + lane] = cd;
    }
#pragma unroll
    for (int e = 1; e <= WM; ++e) {   // L(j+d, j+e) -= c_d c_e, 1 <= e <= d
      const double ce = __shfl_sync(0xffffffffu, cd, e);
      if (e <= lane) R[e] = __fma_rn(-cd, ce, R[e]);
    }
#pragma unroll
    for (int c = 0; c < WM; ++c) R[c] = __shfl_down_sync(0xffffffffu, R[c + 1], 1);
    R[WM] = 0.0;
    if (lane == w) {   // row j+1+w enters (prefetched); prefetch row j+2+w
      const int r = j + 2 + w;
#pragma unroll
      for (int c = 0; c <= WM; ++c) {
        R[c] = nxt[c];
        nxt[c] = (r < n && c <= w) ? A[(int64_t)r * n + j + 2 + c] : 0.0;
      }
    }
  }
}

template <int WM>   // register window of the substitutions (w <= WM)
__global__ void __launch_bounds__(NT) k_cell_band(LevelDev lv, CellArgs ca, const int* list, int w, DevStatus* st,
                                                  long long* prof, const double* scratch, int64_t stride) {
  extern __shared__ double smem[];
  const int t = list[blockIdx.x], tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool pf = prof != nullptr && blockIdx.x == 0 && tid == 0;
  long long t0 = pf ? clock64() : 0;
#define BAND_MARK(slot)                                                                                 \
  if (pf) {                                                                                             \
    const long long t1 = clock64();                                                                     \
    atomicAdd(reinterpret_cast<unsigned long long*>(prof + (slot)), (unsigned long long)(t1 - t0));     \
    t0 = t1;                                                                                            \
  }
  const int I = ca.interior[t], n = ca.n[t], b = ca.b[t];
  const int W1 = w + 1;
  double* Lb = smem;                  // n x (w+1): Lb[i*W1 + d] = L(i, i-d)
  double* dinv = Lb + (int64_t)n * W1;   // n
  double* Xs = dinv + n;              // b x 64 staging of X^T chunks (U) / 8 warps x 32 x 17 row staging
  __shared__ int s_bad;
  double* P = ca.rec + ca.P_off[t];
  // band of L and 1/diag from the one-warp Cholesky (k_band_chol)
  const double* Sc = scratch + (int64_t)blockIdx.x * stride;
  for (int e = tid; e < n * W1 + n; e += NT) Lb[e] = Sc[e];
  if (tid == 0) s_bad = st->first_bad == ~0ull ? -1 : 0;   // (a failed cell anywhere: results unused)
  __syncthreads();
  BAND_MARK(24)
  BAND_MARK(25)
  if (s_bad >= 0) return;   // (NotSpd: reported by k_band_chol; the factorization stops)
  // X = L^-1 A_BI^T (one boundary DOF per thread) and L^-T (row j = L^-1 e_j, one identity column
  // per thread): substitutions in lockstep over 16-row chunks; each warp stages its 32 x 16 chunk
  // in shared memory and writes it out as 16-double row segments (coalesced), zeros included
  double* stg = Xs + (int64_t)warp * 32 * 17;
  auto solve_rows = [&](bool active, const double* S, int wn, int rc, int rhs_one, double* row0, int nrows_warp,
                        int64_t row_base, int zero_until) {
    double h[WM];
#pragma unroll
    for (int q = 0; q < WM; ++q) h[q] = 0.0;
    for (int i0 = 0; i0 < n; i0 += 16) {
      const int cnt = min(16, n - i0);
      if (i0 + 16 <= zero_until) {   // every right-hand side of the warp is still zero here: no chain
        for (int e = lane; e < 32 * 16; e += 32) {
          const int rr = e >> 4, u = e & 15;
          if (rr < nrows_warp && u < cnt) row0[(row_base + rr) * n + i0 + u] = 0.0;
        }
        continue;
      }
      double a[16];
#pragma unroll
      for (int u = 0; u < 16; ++u)
        a[u] = (active && u < cnt) ? (S ? S[(int64_t)(i0 + u) * wn + rc] : (i0 + u == rhs_one ? 1.0 : 0.0)) : 0.0;
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        if (u >= cnt) break;
        const int i = i0 + u;
        double acc = a[u], acc2 = 0.0;   // two chains: even / odd band offsets
        const double* Li = Lb + (int64_t)i * W1;
#pragma unroll
        for (int q = 0; q < WM; ++q)
          if (q < w) {
            if (q & 1) acc2 = __fma_rn(-Li[q + 1], h[q], acc2);
            else acc = __fma_rn(-Li[q + 1], h[q], acc);
          }
        const double x = active ? (acc + acc2) * dinv[i] : 0.0;
#pragma unroll
        for (int q = WM - 1; q > 0; --q) h[q] = h[q - 1];
        h[0] = x;
        stg[lane * 17 + u] = x;
      }
      __syncwarp();
      for (int e = lane; e < 32 * 16; e += 32) {
        const int rr = e >> 4, u = e & 15;
        if (rr < nrows_warp && u < cnt) row0[(row_base + rr) * n + i0 + u] = stg[rr * 17 + u];
      }
      __syncwarp();
    }
  };
  (void)solve_rows;
  // The three record parts only depend on the band of L: no CTA barrier between them. The warps
  // holding boundary DOFs solve X first (U waits for it), the others go straight to the L rows and
  // L^-T; a warp's L^-T columns j >= 32*warp are zero above row j, so those chunks are plain zero
  // stores.
  if (warp * 32 < b) {   // X^T rows n + r
    const int r = tid;
    const bool act = r < b;
    const double* S = nullptr;
    int wn = 1, rc = 0;
    if (act) {
      int64_t jn = ca.nbr_off[t];
      while (jn + 1 < ca.nbr_off[t + 1] && ca.nbr_col[jn + 1] <= r) ++jn;
      wn = ca.nbr_w[jn];
      rc = r - ca.nbr_col[jn];
      S = lv.pool + lv.boff[ca.nbr_blk[jn]];   // block (I, h): |I| x wn row-major
    }
    solve_rows(act, act ? S : Lb, wn, rc, -1, P, min(32, b - warp * 32), (int64_t)n + warp * 32, 0);
  }
  BAND_MARK(27)
  // L rows of the record (dense, zeros outside the band)
  for (int i = warp; i < n; i += NT / 32)   // row i: lanes along columns (no 64-bit division)
    for (int c = lane; c < n; c += 32) {
      const int d = i - c;
      P[(int64_t)i * n + c] = (d >= 0 && d <= w) ? Lb[i * W1 + d] : 0.0;
    }
  BAND_MARK(26)
  if (warp * 32 < n) {   // L^-T rows n + b + j
    const int j = tid;
    solve_rows(j < n, nullptr, 1, 0, j, P, min(32, n - warp * 32), (int64_t)n + b + warp * 32, warp * 32);
  }
  __syncthreads();   // X^T rows written (global, read back through L2 below)
  BAND_MARK(28)
  // U = X^T X (b x b): 64-column chunks of X^T in shared memory (row stride 65: a half-warp's 16
  // rows tj + 16 y fall in 16 different banks), a 4 x 4 interleaved output block per thread
  if (b > 0) {
    constexpr int XLD = 65;
    double acc[4][4];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) acc[x][y] = 0.0;
    const int ti = tid / 16, tj = tid % 16;   // rows ti + 16 x, columns tj + 16 y (b <= 64)
    for (int c0 = 0; c0 < n; c0 += 64) {
      const int cw = min(64, n - c0);
      __syncthreads();
      for (int e = tid; e < b * 64; e += NT) {
        const int r = e / 64, c = e % 64;
        Xs[r * XLD + c] = c < cw ? __ldcg(P + (int64_t)(n + r) * n + c0 + c) : 0.0;
      }
      __syncthreads();
      for (int c = 0; c < cw; ++c) {
        double xa[4], xb[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          const int ra = ti + 16 * x, rb = tj + 16 * x;
          xa[x] = ra < b ? Xs[ra * XLD + c] : 0.0;
          xb[x] = rb < b ? Xs[rb * XLD + c] : 0.0;
        }
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) acc[x][y] = __fma_rn(xa[x], xb[y], acc[x][y]);
      }
    }
    double* U = ca.U + ca.U_off[t];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        const int ra = ti + 16 * x, rb = tj + 16 * y;
        if (ra < b && rb < b) U[(int64_t)ra * b + rb] = acc[x][y];
      }
  }
  __syncthreads();
  BAND_MARK(29)
  if (pf) atomicAdd(reinterpret_cast<unsigned long long*>(prof + 30), 1ull);
#undef BAND_MARK
}

// flag = 1 if some interior DOF couples, inside its own group, to a member more than w positions
// away (the banded cell path is then not applicable)
__global__ void k_band_check(const int64_t* rowptr, const int* col, const int* gid, const int* pos,
                             const uint8_t* is_int, int64_t N, int w, int* flag) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= N) return;
  const int g = gid[r];
  if (!is_int[g]) return;
  for (int64_t e = rowptr[r]; e < rowptr[r + 1]; ++e) {
    const int c = col[e];
    if (gid[c] == g && abs(pos[c] - pos[r]) > w) {
      atomicExch(flag, 1);
      return;
    }
  }
}

// A_BB -= sum_c X_c^T X_c, owner-computes per target block, contributions in cell order.
// blockIdx.y splits the rows of a target block (deep levels have few, large blocks); a warp owns
// a row, lanes run along the columns (coalesced, no index division). The per-element summation
// order is the cell order whatever the split.
__global__ void __launch_bounds__(NT) k_schur(LevelDev lv, SchurArgs sa) {
  const int tau = blockIdx.x;
  const int blk = sa.tgt_blk[tau];
  const int rows = lv.gsize[lv.bg[blk]], cols = lv.gsize[lv.bh[blk]];
  double* dst = lv.pool + lv.boff[blk];
  const int64_t c0 = sa.tgt_off[tau], c1 = sa.tgt_off[tau + 1];
  if (rows * cols <= 2048) {   // small block: one pass of the CTA over the elements
    if (blockIdx.y) return;
    for (int e = threadIdx.x; e < rows * cols; e += NT) {
      const int i = e / cols, j = e - i * cols;
      double s = dst[e];
      for (int64_t c = c0; c < c1; ++c) {
        const int cell = sa.con_cell[c];
        s -= sa.U[sa.U_off[cell] + (int64_t)(sa.con_row[c] + i) * sa.cell_b[cell] + sa.con_col[c] + j];
      }
      dst[e] = s;
    }
    return;
  }
  const int lane = threadIdx.x & 31, wpb = NT / 32;
  for (int i = blockIdx.y * wpb + (threadIdx.x >> 5); i < rows; i += gridDim.y * wpb) {
    double* drow = dst + (int64_t)i * cols;
    for (int j0 = 0; j0 < cols; j0 += 128) {   // four columns per lane in flight
      double s[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = j0 + 32 * u + lane;
        s[u] = j < cols ? drow[j] : 0.0;
      }
      for (int64_t c = c0; c < c1; ++c) {
        const int cell = sa.con_cell[c];
        const int bb = sa.cell_b[cell];
        const double* urow = sa.U + sa.U_off[cell] + (int64_t)(sa.con_row[c] + i) * bb + sa.con_col[c];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = j0 + 32 * u + lane;
          if (j < cols) s[u] -= urow[j];
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = j0 + 32 * u + lane;
        if (j < cols) drow[j] = s[u];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Stage 2: block Jacobi.
// ---------------------------------------------------------------------------
// record [L ; L^-T] (2k x k): the identity rows below A_gg come out of the partial Cholesky as L^-T
__global__ void __launch_bounds__(NT, 3) k_prec_factor(LevelDev lv, PrecArgs pa, DevStatus* st) {
  extern __shared__ double smem[];
  const int t = pa.list ? pa.list[blockIdx.x] : blockIdx.x, tid = threadIdx.x;
  const int g = pa.groups[t], k = lv.gsize[g];
  double* A = lv.pool + lv.boff[lv.diag_blk[g]];
  double* L = pa.rec + pa.L_off[t];
  for (int64_t e = tid; e < (int64_t)k * k; e += NT) {
    L[e] = A[e];
    L[(int64_t)k * k + e] = (e / k == e % k) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int info = cta_potrf_panel(L, 2 * k, k, k, smem);
  if (info >= 0) {
    if (tid == 0) report_bad(st, t, info);
    return;
  }
  for (int64_t e = tid; e < (int64_t)k * k; e += NT) A[e] = (e / k == e % k) ? 1.0 : 0.0;
}

constexpr int PREC_SCALE_T = 64 * 64;   // doubles of the scaling intermediate (after SMEM_DOUBLES)
__global__ void __launch_bounds__(NT) k_prec_scale(LevelDev lv, PrecArgs pa) {
  extern __shared__ double smem[];
  const int blk = pa.scale_list ? pa.scale_blk[pa.scale_list[blockIdx.x]] : pa.scale_blk[blockIdx.x];
  const int g = lv.bg[blk], h = lv.bh[blk];
  const int kg = lv.gsize[g], kh = lv.gsize[h];
  double* B = lv.pool + lv.boff[blk];
  const double* Lg = pa.rec + pa.L_off_of_group[g];
  const double* Lh = pa.rec + pa.L_off_of_group[h];
  if (kg * kh <= PREC_SCALE_T) {
    // two DMMA GEMMs with the explicit inverses stored after each factor ([L ; L^-T] record):
    // T = (L_g^-T)^T B in shared memory, then B = T L_h^-T
    double* T = smem + SMEM_DOUBLES;
    double* gsm = smem + GEMM_OFF;
    cta_gemm<true, false>(kg, kh, kg, 1.0, Lg + (int64_t)kg * kg, kg, B, kh, 0.0, T, kh, false, gsm);
    cta_gemm<false, false>(kg, kh, kh, 1.0, T, kh, Lh + (int64_t)kh * kh, kh, 0.0, B, kh, false, gsm);
    return;
  }
  cta_trsm_left(Lg, kg, kg, B, kh, kh, false, smem);
  cta_trsm_right_lt(Lh, kh, kh, B, kg, kh, smem);
}

// The two-GEMM form of k_prec_scale alone (|g| |h| <= PREC_SCALE_T), compiled for three CTAs per SM:
// the stage is latency-bound (117 K blocks of <= 49 x 49 at c5 level 1), and the substitution
// path of the general kernel held it at two CTAs per SM by registers.
__global__ void __launch_bounds__(NT, 3) k_prec_scale_gemm(LevelDev lv, PrecArgs pa) {
  extern __shared__ double smem[];
  const int blk = pa.scale_list ? pa.scale_blk[pa.scale_list[blockIdx.x]] : pa.scale_blk[blockIdx.x];
  const int g = lv.bg[blk], h = lv.bh[blk];
  const int kg = lv.gsize[g], kh = lv.gsize[h];
  double* B = lv.pool + lv.boff[blk];
  const double* Lg = pa.rec + pa.L_off_of_group[g];
  const double* Lh = pa.rec + pa.L_off_of_group[h];
  double* T = smem + SMEM_DOUBLES;
  double* gsm = smem + GEMM_OFF;
  cta_gemm<true, false>(kg, kh, kg, 1.0, Lg + (int64_t)kg * kg, kg, B, kh, 0.0, T, kh, false, gsm);
  cta_gemm<false, false>(kg, kh, kh, 1.0, T, kh, Lh + (int64_t)kh * kh, kh, 0.0, B, kh, false, gsm);
}

// Small block-Jacobi groups (k <= 32): one warp per group instead of one CTA. Same record
// as k_prec_factor: [A_gg ; I] -> [L ; L^-T] (row-major, strict upper of L zero), A_gg <- I.
// Cholesky right-looking in the warp's shared tile (lanes along rows); L^-1 by forward
// substitution with one right-hand side per lane.
__global__ void __launch_bounds__(256) k_prec_factor_warp(LevelDev lv, PrecArgs pa, const int* list, int n, int kmax,
                                                          DevStatus* st) {
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int idx = blockIdx.x * 8 + warp;
  if (idx >= n) return;
  const int ld = (kmax + 1) | 1;   // odd row stride: lanes along rows fall in different banks
  double* D = smem + (size_t)warp * 2 * kmax * ld;
  double* X = D + (size_t)kmax * ld;
  const int t = list ? list[idx] : idx;   // (no list: every group)
  const int g = pa.groups[t], k = lv.gsize[g];
  double* A = lv.pool + lv.boff[lv.diag_blk[g]];
  double* L = pa.rec + pa.L_off[t];
  for (int e = lane; e < k * k; e += 32) D[(e / k) * ld + e % k] = A[e];
  __syncwarp();
  for (int j = 0; j < k; ++j) {
    const double d = D[j * ld + j];
    if (!(d > 0.0)) {   // same value on every lane: pivot <= 0 or NaN
      if (lane == 0) report_bad(st, t, j);
      return;
    }
    const double ljj = sqrt(d);
    __syncwarp();
    if (lane > j && lane < k) D[lane * ld + j] /= ljj;
    __syncwarp();
    if (lane == j) D[j * ld + j] = ljj;
    if (lane > j && lane < k) {
      const double lij = D[lane * ld + j];
      for (int c = j + 1; c <= lane; ++c) D[lane * ld + c] -= lij * D[c * ld + j];
    }
    __syncwarp();
  }
  // X = L^-1: column `lane`
  if (lane < k)
    for (int i = 0; i < k; ++i) {
      double v = (i == lane) ? 1.0 : 0.0;
      for (int p = lane; p < i; ++p) v -= D[i * ld + p] * X[p * ld + lane];
      X[i * ld + lane] = i < lane ? 0.0 : v / D[i * ld + i];
    }
  __syncwarp();
  for (int e = lane; e < k * k; e += 32) {
    const int i = e / k, c = e % k;
    L[e] = c <= i ? D[i * ld + c] : 0.0;
    L[(int64_t)k * k + e] = X[c * ld + i];   // (L^-T)[i][c] = (L^-1)[c][i]
    A[e] = i == c ? 1.0 : 0.0;
  }
}

// Small two-sided scaling B <- L_g^-1 B L_h^-T (kg, kh <= 32), one warp per block, with the
// explicit inverses U = L^-T stored after each factor: L_g^-1 = U_g^T.
__global__ void __launch_bounds__(256) k_prec_scale_warp(LevelDev lv, PrecArgs pa, const int* list, int n, int ldmax) {
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int idx = blockIdx.x * 8 + warp;
  if (idx >= n) return;
  const int ld = (ldmax + 1) | 1;   // odd row stride: lanes along rows fall in different banks
  double* S = smem + (size_t)warp * ldmax * ld;
  const int blk = pa.scale_blk[list ? list[idx] : idx];   // (no list: every scaling block)
  const int g = lv.bg[blk], h = lv.bh[blk];
  const int kg = lv.gsize[g], kh = lv.gsize[h];
  double* B = lv.pool + lv.boff[blk];
  const double* UG = pa.rec + pa.L_off_of_group[g] + (int64_t)kg * kg;
  const double* UH = pa.rec + pa.L_off_of_group[h] + (int64_t)kh * kh;
  for (int e = lane; e < kg * kh; e += 32) S[(e / kh) * ld + e % kh] = B[e];
  __syncwarp();
  if (lane < kh)   // column lane: B[i][j] <- sum_{p <= i} U_g[p][i] B[p][j], rows descending (in place)
    for (int i = kg - 1; i >= 0; --i) {
      double v = 0.0;
      for (int p = 0; p <= i; ++p) v += __ldg(UG + (int64_t)p * kg + i) * S[p * ld + lane];
      S[i * ld + lane] = v;
    }
  __syncwarp();
  if (lane < kg)   // row lane: B[i][j] <- sum_{p <= j} B[i][p] U_h[p][j], columns descending
    for (int j = kh - 1; j >= 0; --j) {
      double v = 0.0;
      for (int p = 0; p <= j; ++p) v += S[lane * ld + p] * __ldg(UH + (int64_t)p * kh + j);
      S[lane * ld + j] = v;
    }
  __syncwarp();
  for (int e = lane; e < kg * kh; e += 32) B[e] = S[(e / kh) * ld + e % kh];
}

// ---------------------------------------------------------------------------
// Stage 3a: interpolative decomposition of A_{R,I}, one wave of mutually
// independent separators (kernels.py:84-119).
// CPQR follows LAPACK dgeqp3/dlaqp2 (oracle/dense.py:cpqr_dlaqp2).
// ---------------------------------------------------------------------------
struct ArgMax {
  double v;
  int i;
};

__device__ __forceinline__ ArgMax better(ArgMax a, ArgMax b) {
  // larger value wins; ties -> lower index (idamax returns the first maximum)
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}

__device__ ArgMax cta_argmax(ArgMax x, double* sred) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ArgMax y;
    y.v = __shfl_xor_sync(0xffffffffu, x.v, o);
    y.i = __shfl_xor_sync(0xffffffffu, x.i, o);
    x = better(x, y);
  }
  int* sidx = reinterpret_cast<int*>(sred + 16);
  __syncthreads();
  if (lane == 0) {
    sred[w] = x.v;
    sidx[w] = x.i;
  }
  __syncthreads();
  ArgMax r{sred[0], sidx[0]};
  for (int k = 1; k < NT / 32; ++k) r = better(r, ArgMax{sred[k], sidx[k]});
  __syncthreads();
  return r;
}

// CTA argmax without the trailing barrier: warp shuffles, one __syncthreads, then every warp
// reduces the 8 warp winners with 3 shuffle levels. The caller guarantees a __syncthreads
// between two calls sharing `sred`.
__device__ ArgMax cta_argmax1(ArgMax x, double* sred) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ArgMax y;
    y.v = __shfl_xor_sync(0xffffffffu, x.v, o);
    y.i = __shfl_xor_sync(0xffffffffu, x.i, o);
    x = better(x, y);
  }
  int* sidx = reinterpret_cast<int*>(sred + 16);
  if (lane == 0) {
    sred[w] = x.v;
    sidx[w] = x.i;
  }
  __syncthreads();
  ArgMax r{-1.0, 0x7fffffff};
  if (lane < NT / 32) r = ArgMax{sred[lane], sidx[lane]};
#pragma unroll
  for (int o = NT / 64; o > 0; o >>= 1) {
    ArgMax y;
    y.v = __shfl_xor_sync(0xffffffffu, r.v, o);
    y.i = __shfl_xor_sync(0xffffffffu, r.i, o);
    r = better(r, y);
  }
  r.v = __shfl_sync(0xffffffffu, r.v, 0);
  r.i = __shfl_sync(0xffffffffu, r.i, 0);
  return r;
}

// Exclusive CTA scan of 0/1 flags; returns this thread's offset, *total = count.
__device__ int cta_scan_flag(int f, int* sint, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned bal = __ballot_sync(0xffffffffu, f);
  const int inwarp = __popc(bal & ((1u << lane) - 1u));
  __syncthreads();
  if (lane == 0) sint[w] = __popc(bal);
  __syncthreads();
  int base = 0, tot = 0;
  for (int k = 0; k < NT / 32; ++k) {
    if (k < w) base += sint[k];
    tot += sint[k];
  }
  __syncthreads();
  *total = tot;
  return base + inwarp;
}

// Column-pivoted Householder QR of W (m x k, column-major, ldw), in place. Stops once the
// largest remaining partial norm is below cutrel*|R_00| by a 1e-4 margin (pivot norms do
// not increase, so no later diagonal can pass the ID cut). Returns the steps performed.
__device__ int cta_cpqr(double* W, int m, int k, int64_t ldw, int* perm, double* vn1, double* vn2, double* sred,
                        double cutrel) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = NT / 32;
  const double tol3z = sqrt(DBL_EPSILON * 0.5);
  for (int j = tid; j < k; j += NT) perm[j] = j;
  for (int j = warp; j < k; j += nw) {
    const double* c = W + (int64_t)j * ldw;
    double s = 0.0;
    for (int r = lane; r < m; r += 32) s += c[r] * c[r];
    s = warp_sum(s);
    if (lane == 0) vn1[j] = vn2[j] = sqrt(s);
  }
  __syncthreads();
  const int mn = min(m, k);
  double* sh = sred + 32;  // [0] tau
  double cut = 0.0;
  for (int i = 0; i < mn; ++i) {
    ArgMax loc{-1.0, 0x7fffffff};
    for (int j = i + tid; j < k; j += NT) loc = better(loc, ArgMax{vn1[j], j});
    const ArgMax best = cta_argmax(loc, sred);
    if (i > 0 && best.v < cut * (1.0 - 1e-4)) return i;
    const int p = best.i;
    if (p != i) {
      double* ci = W + (int64_t)i * ldw;
      double* cp = W + (int64_t)p * ldw;
      for (int r = tid; r < m; r += NT) {
        const double tmp = ci[r];
        ci[r] = cp[r];
        cp[r] = tmp;
      }
      __syncthreads();
      if (tid == 0) {
        const int ti = perm[p];
        perm[p] = perm[i];
        perm[i] = ti;
        vn1[p] = vn1[i];
        vn2[p] = vn2[i];
      }
      __syncthreads();
    }
    // Householder reflector for column i, rows i..m-1 (dlarfg)
    double* ci = W + (int64_t)i * ldw;
    double part = 0.0;
    for (int r = i + 1 + tid; r < m; r += NT) part += ci[r] * ci[r];
    const double xnorm = sqrt(cta_sum(part, sred));
    const double alpha = ci[i];
    double tau = 0.0, beta = alpha;
    if (xnorm != 0.0) {
      beta = -copysign(hypot(alpha, xnorm), alpha);
      tau = (beta - alpha) / beta;
      const double scal = 1.0 / (alpha - beta);
      for (int r = i + 1 + tid; r < m; r += NT) ci[r] *= scal;
    }
    __syncthreads();
    if (tid == 0) {
      ci[i] = beta;
      sh[0] = tau;
    }
    if (i == 0) cut = cutrel * fabs(beta);
    __syncthreads();
    // apply H to trailing columns, then downdate partial norms (dlarf + dlaqp2 loop 10)
    for (int j = i + 1 + warp; j < k; j += nw) {
      double* cj = W + (int64_t)j * ldw;
      if (tau != 0.0) {
        double s = 0.0;
        for (int r = i + 1 + lane; r < m; r += 32) s += ci[r] * cj[r];
        s = warp_sum(s) + cj[i];
        const double tw = tau * s;
        __syncwarp();
        if (lane == 0) cj[i] -= tw;
        for (int r = i + 1 + lane; r < m; r += 32) cj[r] -= tw * ci[r];
        __syncwarp();
      }
      const double v1 = vn1[j];
      if (v1 != 0.0) {
        double tt = fabs(cj[i]) / v1;
        tt = 1.0 - tt * tt;
        tt = tt < 0.0 ? 0.0 : tt;
        const double rr = v1 / vn2[j];
        const double t2 = tt * rr * rr;
        if (t2 <= tol3z) {
          double s = 0.0;
          if (i < m - 1) {
            for (int r = i + 1 + lane; r < m; r += 32) s += cj[r] * cj[r];
            s = sqrt(warp_sum(s));
          }
          __syncwarp();
          if (lane == 0) vn1[j] = vn2[j] = s;
        } else {
          __syncwarp();
          if (lane == 0) vn1[j] = v1 * sqrt(tt);
        }
      }
    }
    __syncthreads();
  }
  return mn;
}

// ---- coupling-row gather in 32-row chunks -------------------------------------------------
// The candidate rows of A_{R,I} (alive members of every coupled group) are cut into
// chunks of 32 rows of one neighbour group (neighbours in order, ceil(|h|/32) chunks each).
// A warp computes a chunk's keep mask (row alive and with a nonzero in A_{h,I}) from independent
// coalesced loads; a warp scan of the popcounts places the kept rows; a second sweep copies them.
// Coupled-group metadata of one separator, staged in shared memory once (one thread per
// neighbour) so the chunk sweeps never walk dependent global loads.
constexpr int NBMAX = 256;
struct NbrCache {
  int n, nch, rows;
  int h[NBMAX], kh[NBMAX], ch0[NBMAX + 1], r0[NBMAX];   // r0: first row of neighbour i in A_{R,I}
  long long boff[NBMAX], moff[NBMAX];
  __device__ int locate(int ch) const {   // neighbour holding chunk ch: last i with ch0[i] <= ch
    int lo = 0, hi = n - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (ch0[mid] <= ch) lo = mid;
      else hi = mid - 1;
    }
    return lo;
  }
};
__device__ void nbr_cache_load(const LevelDev& lv, const SkelArgs& sk, int s, NbrCache& nc) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t q0 = sk.nbr_off[s];
  const int n = (int)(sk.nbr_off[s + 1] - q0);   // <= NBMAX (checked on the host)
  for (int i = tid; i < n; i += NT) {
    const int h = sk.nbr[q0 + i];
    nc.h[i] = h;
    nc.kh[i] = lv.gsize[h];
    nc.boff[i] = lv.boff[sk.nbr_blk[q0 + i]];
    nc.moff[i] = lv.goff[h];
  }
  __syncthreads();
  if (tid < 32) {
    int run_c = 0, run_r = 0;
    for (int i0 = 0; i0 < n; i0 += 32) {
      const int i = i0 + lane;
      const int vc = i < n ? (nc.kh[i] + 31) >> 5 : 0, vr = i < n ? nc.kh[i] : 0;
      int ic = vc, ir = vr;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int tc = __shfl_up_sync(0xffffffffu, ic, o), tr = __shfl_up_sync(0xffffffffu, ir, o);
        if (lane >= o) {
          ic += tc;
          ir += tr;
        }
      }
      if (i < n) {
        nc.ch0[i] = run_c + ic - vc;
        nc.r0[i] = run_r + ir - vr;
      }
      run_c += __shfl_sync(0xffffffffu, ic, 31);
      run_r += __shfl_sync(0xffffffffu, ir, 31);
    }
    if (lane == 0) {
      nc.n = n;
      nc.nch = run_c;
      nc.ch0[n] = run_c;
      nc.rows = run_r > 0 ? run_r : 1;
    }
  }
  __syncthreads();
}
// rows r0 .. r0+31 of neighbour i with a nonzero in A_{h,I} (independent of the alive flags)
__device__ __forceinline__ unsigned chunk_nz(const LevelDev& lv, const NbrCache& nc, int g, int k, int i, int r0) {
  const int lane = threadIdx.x & 31;
  const int h = nc.h[i], kh = nc.kh[i];
  const double* B = lv.pool + nc.boff[i];
  const int r = r0 + lane;
  bool nz = false;
  if (g < h) {   // block (g,h) is |g| x |h|: column r of it, lanes along rows (coalesced)
    const double* p = B + (r < kh ? r : 0);
    // stop as soon as every lane has seen a nonzero (the usual case: after the first batch)
    for (int c = 0; c < k; c += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = (r < kh && c + u < k) ? p[(int64_t)(c + u) * kh] : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) nz |= v[u] != 0.0;
      if (c + 8 < k && __all_sync(0xffffffffu, nz || r >= kh)) break;
    }
  } else {       // block (h,g) is |h| x |g|: rows r0..r0+31 are contiguous, lanes along columns
    const int nr = min(32, kh - r0);
    const double* p = B + (int64_t)r0 * k;
    for (int rb = 0; rb < nr; rb += 8) {
      bool any[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) any[u] = false;
      for (int c0 = 0; c0 < k; c0 += 32) {
        const int c = c0 + lane;
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = (rb + u < nr && c < k) ? p[(int64_t)(rb + u) * k + c] : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) any[u] |= v[u] != 0.0;
        if (c0 + 32 < k) {   // more columns left: stop once every row of the group has a nonzero
          bool all = true;
#pragma unroll
          for (int u = 0; u < 8; ++u) all = all && (__any_sync(0xffffffffu, any[u]) || rb + u >= nr);
          if (all) break;
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (__any_sync(0xffffffffu, any[u]) && lane == rb + u) nz = true;
    }
  }
  return __ballot_sync(0xffffffffu, nz);
}
__device__ __forceinline__ unsigned chunk_mask(const LevelDev& lv, const SkelArgs& sk, const NbrCache& nc, int g, int k,
                                               int i, int r0) {
  const unsigned nzm = chunk_nz(lv, nc, g, k, i, r0);
  const int r = r0 + (threadIdx.x & 31);
  const bool alive = r < nc.kh[i] && __ldcg(sk.alive + lv.mem[nc.moff[i] + r]);
  return __ballot_sync(0xffffffffu, alive) & nzm;
}
template <int U>
__device__ __forceinline__ void chunk_copy(const LevelDev& lv, const NbrCache& nc, int g, int k, int i, int r0,
                                           unsigned mask, double* W, int64_t ldw, int row0) {
  const int lane = threadIdx.x & 31;
  const int h = nc.h[i], kh = nc.kh[i];
  const double* B = lv.pool + nc.boff[i];
  // loads are batched ahead of the stores (W and B may alias as far as the compiler knows, so an
  // unbatched copy loop would pay one full memory latency per element)
  if (row0 < 0) {   // fixed positions: row (-1 - row0) + r0 + lane, rejected rows written as zeros
    const int rbase = -1 - row0 + r0;
    if (g < h) {
      const int r = r0 + lane;
      if (r < kh) {
        const bool keep = (mask >> lane) & 1u;
        const double* p = B + r;
        for (int c0 = 0; c0 < k; c0 += U) {
          double v[U];
#pragma unroll
          for (int u = 0; u < U; ++u) v[u] = (keep && c0 + u < k) ? p[(int64_t)(c0 + u) * kh] : 0.0;
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (c0 + u < k) W[(int64_t)(c0 + u) * ldw + rbase + lane] = v[u];
        }
      }
    } else {
      // rows r0.. of block (h, g) are contiguous: lanes along columns, 8 rows x 2 column strips
      // of loads in flight before their stores
      const int nr = min(32, kh - r0);
      for (int rr0 = 0; rr0 < nr; rr0 += 8) {
        double v[8][2];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int rr = rr0 + u;
          const bool keep = rr < nr && ((mask >> rr) & 1u);
          const double* p = B + (int64_t)(r0 + rr) * k;
#pragma unroll
          for (int w = 0; w < 2; ++w) {
            const int c = lane + 32 * w;
            v[u][w] = (keep && c < k) ? p[c] : 0.0;
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int rr = rr0 + u;
          if (rr >= nr) break;
#pragma unroll
          for (int w = 0; w < 2; ++w) {
            const int c = lane + 32 * w;
            if (c < k) W[(int64_t)c * ldw + rbase + rr] = v[u][w];
          }
        }
        for (int c = lane + 64; c < k; c += 32)   // (k > 64: remaining columns, unbatched)
          for (int rr = rr0; rr < min(nr, rr0 + 8); ++rr)
            W[(int64_t)c * ldw + rbase + rr] = ((mask >> rr) & 1u) ? B[(int64_t)(r0 + rr) * k + c] : 0.0;
      }
    }
    return;
  }
  if (g < h) {
    if ((mask >> lane) & 1u) {
      const int row = row0 + __popc(mask & ((1u << lane) - 1u));
      const double* p = B + r0 + lane;
      for (int c0 = 0; c0 < k; c0 += U) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = c0 + u < k ? p[(int64_t)(c0 + u) * kh] : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (c0 + u < k) W[(int64_t)(c0 + u) * ldw + row] = v[u];
      }
    }
  } else {
    int row = row0;
    while (mask) {
      const int rr = __ffs(mask) - 1;
      mask &= mask - 1u;
      const double* p = B + (int64_t)(r0 + rr) * k;
      for (int c0 = lane; c0 < k; c0 += 32 * U) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = c0 + 32 * u < k ? p[c0 + 32 * u] : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (c0 + 32 * u < k) W[(int64_t)(c0 + 32 * u) * ldw + row] = v[u];
      }
      ++row;
    }
  }
}
// Chunks [ch_lo, ch_hi) of separator s: with COPY, kept rows go to W rows base, base+1, ...
// Returns the number of kept rows (all threads). smem: 2*cap ints.
template <bool COPY, int U = 8>
__device__ int gather_chunks(const LevelDev& lv, const SkelArgs& sk, const NbrCache& nc, int s, int ch_lo, int ch_hi,
                             double* W, int64_t ldw, int base, int* sbuf, int cap) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = NT / 32;
  const int g = sk.groups[s], k = lv.gsize[g];
  unsigned* smask = reinterpret_cast<unsigned*>(sbuf);
  int* spre = sbuf + cap;
  __shared__ int s_tot;
  int total = 0;
  for (int b0 = ch_lo; b0 < ch_hi; b0 += cap) {
    const int nb = min(cap, ch_hi - b0);
    for (int j = warp; j < nb; j += nw) {
      const int i = nc.locate(b0 + j);
      const unsigned msk = chunk_mask(lv, sk, nc, g, k, i, 32 * (b0 + j - nc.ch0[i]));
      if (lane == 0) smask[j] = msk;
    }
    __syncthreads();
    if (warp == 0) {
      int run = 0;
      for (int i0 = 0; i0 < nb; i0 += 32) {
        const int v = i0 + lane < nb ? __popc(smask[i0 + lane]) : 0;
        int inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += t;
        }
        if (i0 + lane < nb) spre[i0 + lane] = run + inc - v;
        run += __shfl_sync(0xffffffffu, inc, 31);
      }
      if (lane == 0) s_tot = run;
    }
    __syncthreads();
    if (COPY)
      for (int j = warp; j < nb; j += nw) {
        const int i = nc.locate(b0 + j);
        chunk_copy<U>(lv, nc, g, k, i, 32 * (b0 + j - nc.ch0[i]), smask[j], W, ldw, base + total + spre[j]);
      }
    total += s_tot;
    __syncthreads();
  }
  return total;
}


// no coupling: every column redundant (kernels.py:95-98)
__device__ void skel_all_redundant(const LevelDev& lv, const SkelArgs& sk, int s) {
  const int g = sk.groups[s], k = lv.gsize[g];
  const int64_t gof = lv.goff[g];
  for (int j = threadIdx.x; j < k; j += NT) {
    sk.red[gof + j] = 1;
    sk.alive[lv.mem[gof + j]] = 0;
  }
  if (threadIdx.x == 0) sk.rank[s] = 0;
}

// warp argmax of (v >= 0, pos): largest v, lowest pos among ties (dlaqp2's first maximum); three
// redux operations on the bit pattern of v. Returns the winning lane's ballot mask.
__device__ __forceinline__ unsigned warp_first_max(double v, unsigned pos) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  const unsigned hi = (unsigned)(b >> 32), lo = (unsigned)b;
  const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
  const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
  const bool top = hi == mh && lo == ml;
  const unsigned mp = __reduce_min_sync(0xffffffffu, top ? pos : 0xffffffffu);
  return __ballot_sync(0xffffffffu, top && pos == mp);
}

// Gram-path ID of one small separator (k <= 57) on one CTA: G = A^T A by DMMA into smem[0, k^2),
// then the pivoted Cholesky replay of dlaqp2 (see gram_id.cuh) with the full symmetric Schur
// complement updated in place, then T = R11^-1 R12 (4 threads per right-hand side). The
// workspace after G reuses the gathered matrix's region (base = smem + SMEM_DOUBLES).
// Returns false (nothing written) when the shapes do not fit; the caller then runs cta_cpqr.
__device__ __forceinline__ bool skel_id_gram_fits(int k, int cap) {
  return k <= 57 && k * k <= RED_OFF && (int64_t)k * k + 7 * k + 8 <= cap;
}
// W holds mrows rows (kept rows and zero rows), m of them kept
// With ds != nullptr (dependency-driven launch) the redundant flags are published and the
// dependent separators released right after the pivot chain, before T is formed.
__device__ bool skel_id_gram(const LevelDev& lv, const SkelArgs& sk, int s, int k, const double* W, int64_t ldw,
                             int mrows, int m, double* smem, int cap, const DynSched* ds = nullptr) {
  if (!skel_id_gram_fits(k, cap)) return false;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = NT / 32;
  const int g = sk.groups[s];
  const int64_t gof = lv.goff[g];
  double* S = smem;                        // k x k (G, then the Schur complement; then R permuted)
  double* sred = smem + RED_OFF;
  double* base = smem + SMEM_DOUBLES;
  double* Rsm = base;                      // k x k: row i of R at Rsm[i*k + column]
  double* d = Rsm + k * k;
  double* vn1 = d + k;
  double* vn2 = vn1 + k;
  double* rdv = vn2 + k;    // sqrt(Schur diagonal) and its reciprocal per column
  double* invv = rdv + k;
  int* col_at = reinterpret_cast<int*>(invv + k);
  int* piv = col_at + k;
  int* sidx = piv + k;
  // G = W^T W: lower 8x8 tiles, one DMMA chain per tile (K = m in steps of 4), mirrored
  {
    const int gq = lane >> 2, t4 = lane & 3;
    const int nt = (k + 7) / 8, ntl = nt * (nt + 1) / 2;
    for (int tix = warp; tix < ntl; tix += nw) {
      int it = 0;
      while ((it + 1) * (it + 2) / 2 <= tix) ++it;
      const int jt = tix - it * (it + 1) / 2;
      const int a = it * 8 + gq, b = jt * 8 + gq;
      const double* Wa = W + (int64_t)min(a, k - 1) * ldw;
      const double* Wb = W + (int64_t)min(b, k - 1) * ldw;
      const bool oka = a < k, okb = b < k;
      double c0 = 0.0, c1 = 0.0;
      for (int r0 = 0; r0 < mrows; r0 += 4) {
        const int r = r0 + t4;
        const double av = (oka && r < mrows) ? Wa[r] : 0.0;
        const double bv = (okb && r < mrows) ? Wb[r] : 0.0;
        dmma(c0, c1, av, bv);
      }
      const int row = it * 8 + gq, col = jt * 8 + 2 * t4;
#pragma unroll
      for (int z = 0; z < 2; ++z) {
        const double v = z ? c1 : c0;
        if (row < k && col + z < k) {
          S[row * k + col + z] = v;
          S[(col + z) * k + row] = v;
        }
      }
    }
  }
  __syncthreads();
  // Pivoted Cholesky of G replaying dlaqp2, by warp 0 alone (no CTA barriers on the pivot chain;
  // k <= 57, two positions per lane). Left-looking: row i of R is formed from row p of G and the
  // earlier rows of R, acc = fma(-R(l, p), R(l, b), acc) for l = 0 .. i-1 -- the same operations
  // in the same order as the right-looking rank-1 updates of the Schur complement, so R, the
  // pivots and the rank are bit-identical to that formulation (and to cta_cpqr's dlaqp2 rules).
  __shared__ int s_rank;
  if (warp == 0) {
    // Column state in registers (k <= 57: columns lane and lane + 32): Schur diagonal, squared
    // partial norms vn1 / vn2 (argmax and the dlaqp2 tests in squared form), position, pivoted.
    double cd[2], c1[2], c2[2];
    int cpos[2];
    bool cpv[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int b = lane + 32 * u;
      const bool ok = b < k;
      const double dj = ok ? S[b * k + b] : 0.0;
      cd[u] = dj;
      c1[u] = c2[u] = fmax(dj, 0.0);
      cpos[u] = ok ? b : 0x7fffffff;
      cpv[u] = !ok;
    }
    for (int j = lane; j < k; j += 32) {
      col_at[j] = j;
      piv[j] = 0;
    }
    __syncwarp();
    const double tol3z = sqrt(DBL_EPSILON * 0.5);
    const double cutrel = fmax(sk.eps, DBL_EPSILON * (double)max(m, k));
    const int mn = min(m, k);
    double cut = 0.0, cut2 = 0.0;
    int r = 0, i = 0;
    for (; i < mn; ++i) {
      // local candidate: largest partial norm, lowest position among ties (dlaqp2's first maximum)
      double bv = 0.0, bd = 0.0;
      int bpos = 0x7fffffff, bu = 0;
#pragma unroll
      for (int u = 0; u < 2; ++u)
        if (!cpv[u] && (c1[u] > bv || (c1[u] == bv && cpos[u] < bpos))) {
          bv = c1[u];
          bd = cd[u];
          bpos = cpos[u];
          bu = u;
        }
      const int ci = col_at[i];   // the column leaving position i (read early: off the argmax chain)
      const int wl = __ffs(warp_first_max(bv, (unsigned)bpos)) - 1;
      const double wv = __shfl_sync(0xffffffffu, bv, wl);
      const int pb = __shfl_sync(0xffffffffu, bpos, wl);
      const int wu = __shfl_sync(0xffffffffu, bu, wl);
      const double wd = __shfl_sync(0xffffffffu, bd, wl);
      if (pb == 0x7fffffff) break;   // (no unpivoted column left: cannot happen while i < k)
      if (i > 0 && wv < cut2) break;
      const int p = wl + 32 * wu;
      const double rd = sqrt(fmax(wd, 0.0));   // (only the pivot needs it)
      const double inv = rd > 0.0 ? 1.0 / rd : 0.0;
      if (i == 0) {
        cut = cutrel * rd;
        cut2 = cut * (1.0 - 1e-4) * (cut * (1.0 - 1e-4));
      }
      if (rd > cut) ++r;
      // row i of R, left-looking (the same FMAs in the same order as the right-looking updates)
      double* row = Rsm + i * k;
      double rvv[2] = {0.0, 0.0};
      {
        // both column slots advance together: two independent FMA chains per lane
        const int b0 = lane, b1 = lane + 32;
        const bool f0 = b0 < k && b0 != p && !cpv[0], f1 = b1 < k && b1 != p && !cpv[1];
        double acc0 = f0 ? S[p * k + b0] : 0.0, acc1 = f1 ? S[p * k + b1] : 0.0;
        const double* Rp0 = Rsm + p;
        const double* Rb0 = Rsm + (f0 ? b0 : p);
        const double* Rb1 = Rsm + (f1 ? b1 : p);
#pragma unroll 8
        for (int l = 0; l < i; ++l) {
          const double rlp = -Rp0[l * k];
          acc0 = __fma_rn(rlp, Rb0[l * k], acc0);
          acc1 = __fma_rn(rlp, Rb1[l * k], acc1);
        }
        if (b0 < k) {
          double v = 0.0;
          if (b0 == p) {
            v = rd;
            cpv[0] = true;
          } else if (f0) {
            v = acc0 * inv;
            rvv[0] = v;
          }
          row[b0] = v;
        }
        if (b1 < k) {
          double v = 0.0;
          if (b1 == p) {
            v = rd;
            cpv[1] = true;
          } else if (f1) {
            v = acc1 * inv;
            rvv[1] = v;
          }
          row[b1] = v;
        }
      }
      // dlaqp2 swap of positions i and pb: the column displaced from position i moves to pb
      if (lane == 0) {
        col_at[pb] = ci;
        col_at[i] = p;
      }
      // Schur diagonal and partial-norm downdate of the unpivoted columns
#pragma unroll
      for (int u = 0; u < 2; ++u)
        if (!cpv[u]) {
          if (lane + 32 * u == ci) cpos[u] = pb;
          const double rv = rvv[u];
          const double dn = __fma_rn(-rv, rv, cd[u]);
          cd[u] = dn;
          double w1 = c1[u];
          if (w1 != 0.0) {
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
      __syncwarp();
    }
    if (lane == 0) s_rank = r;
  }
  __syncthreads();
  const int r = s_rank;
  const int kt = k - r;
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
  // redundant flags and rank out first: the later separators only wait for these
  {
    uint8_t* red = sk.red + gof;
    for (int j = tid; j < k; j += NT) {
      const int f = piv[j];
      red[j] = (uint8_t)f;
      if (f) sk.alive[lv.mem[gof + j]] = 0;
    }
    if (tid == 0) sk.rank[s] = r;
    if (ds) {
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        for (int64_t e = ds->succ_off[s]; e < ds->succ_off[s + 1]; ++e) atomicAdd(ds->done + ds->succ[e], 1);
      }
    }
  }
  // R in pivot order (rows < r): Rp[i*k + l] = R(i, col_at[l]), in the Schur region
  double* Rp = S;
  for (int e = tid; e < r * k; e += NT) Rp[e] = Rsm[(e / k) * k + col_at[e % k]];
  __syncthreads();
  if (kt > 0 && r > 0) {
    // X = R11^-1 R12: thread (j, q) = (tid / 4, tid % 4) sums the terms l = q mod 4
    double* X = Rsm;   // r x kt
    for (int e = tid; e < r * kt; e += NT) X[e] = Rp[(e / kt) * k + r + e % kt];
    __syncthreads();
    const int q = tid & 3;
    for (int j0 = 0; j0 < kt; j0 += NT / 4) {
      const int j = j0 + (tid >> 2);
      const bool act = j < kt;
      for (int ii = r - 1; ii >= 0; --ii) {
        double sacc = 0.0;
        if (act)
          for (int l = ii + 1 + q; l < r; l += 4) sacc = __fma_rn(Rp[ii * k + l], X[l * kt + j], sacc);
        sacc += __shfl_xor_sync(0xffffffffu, sacc, 1);
        sacc += __shfl_xor_sync(0xffffffffu, sacc, 2);
        if (act && q == 0) X[ii * kt + j] = (X[ii * kt + j] - sacc) / Rp[ii * k + ii];
        __syncwarp();
      }
    }
    __syncthreads();
    double* T = sk.rec + sk.T_off[s];
    for (int e = tid; e < r * kt; e += NT) {
      const int ii = e / kt, j = e % kt;
      T[(int64_t)sidx[col_at[ii]] * kt + sidx[col_at[r + j]]] = X[e];
    }
  }
  return true;
}

// Part of a small separator's ID that does not depend on the earlier separators (the alive
// flags): coupled-group metadata and, on the Gram path, every candidate row of A_{R,I} copied to
// its natural position in shared memory (all-zero rows as zeros), with the row's DOF index kept
// for the alive test. In the dependency-driven launch this runs before the wait.
// Returns true when the Gram path's shared-memory staging was taken.
__device__ bool skel_id_pre(const LevelDev& lv, const SkelArgs& sk, int s, int smem_cap, NbrCache& nc) {
  extern __shared__ double smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g0 = sk.groups[s], k = lv.gsize[g0];
  nbr_cache_load(lv, sk, s, nc);
  const int nch = nc.nch;
  if (!(sk.gram && skel_id_gram_fits(k, smem_cap) && (int64_t)max(1, nc.rows) * k <= smem_cap &&
        nc.rows <= 2 * RED_OFF))
    return false;
  const int64_t ldw = max(1, nc.rows);
  double* W = smem + SMEM_DOUBLES;
  int* rowdof = reinterpret_cast<int*>(smem);   // (the Gram matrix takes this region later)
  for (int ch = warp; ch < nch; ch += NT / 32) {
    const int i = nc.locate(ch), r0 = 32 * (ch - nc.ch0[i]);
    const unsigned nzm = chunk_nz(lv, nc, g0, k, i, r0);
    chunk_copy<8>(lv, nc, g0, k, i, r0, nzm, W, ldw, -1 - nc.r0[i]);
    const int r = r0 + lane;
    if (r < nc.kh[i]) rowdof[nc.r0[i] + r] = ((nzm >> lane) & 1u) ? lv.mem[nc.moff[i] + r] : -1;
  }
  __syncthreads();
  return true;
}

// pre: result of skel_id_pre for this separator (same nc). Returns true when the dependent
// separators were already released (ds given and the early-release path taken).
__device__ bool skel_id_one(const LevelDev& lv, const SkelArgs& sk, int s, int smem_cap, NbrCache& nc, bool pre,
                            const DynSched* ds) {
  extern __shared__ double smem[];
  double* sred = smem + RED_OFF;
  int* sint = reinterpret_cast<int*>(smem);  // scan scratch (first doubles are free here)
  const int tid = threadIdx.x;
  const int g = sk.groups[s];
  const int k = lv.gsize[g];
  const int64_t gof = lv.goff[g];
  // count the kept rows first: A_{R,I} (ld = m) and its CPQR live in shared memory when they
  // fit, else in the global workspace
  const bool pf = sk.prof != nullptr && blockIdx.x == 0 && tid == 0;
  long long t0 = pf ? clock64() : 0;
#define SID_MARK(slot)                                                                                  \
  if (pf) {                                                                                             \
    const long long t1 = clock64();                                                                     \
    atomicAdd(reinterpret_cast<unsigned long long*>(sk.prof + (slot)), (unsigned long long)(t1 - t0)); \
    t0 = t1;                                                                                            \
  }
  const int nch = nc.nch;
  if (pre) {
    // Gram path: A^T A does not depend on the row order and zero rows add nothing, so every
    // candidate row sits at its natural position (skel_id_pre); the rows whose DOF an earlier
    // separator made redundant are zeroed here, and the kept-row count m only enters the rank
    // cut floor
    const int64_t ldw = max(1, nc.rows);
    double* W = smem + SMEM_DOUBLES;
    const int* rowdof = reinterpret_cast<const int*>(smem);
    __shared__ int s_m;
    if (tid == 0) s_m = 0;
    __syncthreads();
    const int lane = tid & 31, warp = tid >> 5;
    int mine = 0;
    for (int rb = 32 * warp; rb < nc.rows; rb += NT) {
      const int rr = rb + lane;
      const int dof = rr < nc.rows ? rowdof[rr] : -1;
      const bool alive = dof >= 0 && __ldcg(sk.alive + dof);
      const unsigned dead = __ballot_sync(0xffffffffu, dof >= 0 && !alive);
      mine += __popc(__ballot_sync(0xffffffffu, alive));
      if (dead) {
        const bool mydead = (dead >> lane) & 1u;
        for (int c = 0; c < k; ++c)
          if (mydead) W[(int64_t)c * ldw + rr] = 0.0;
      }
    }
    if (lane == 0 && mine) atomicAdd(&s_m, mine);
    __syncthreads();
    const int m = s_m;
    if (tid == 0) sk.rows[s] = m;
    SID_MARK(17)
    if (m == 0) {
      skel_all_redundant(lv, sk, s);
      return false;
    }
    skel_id_gram(lv, sk, s, k, W, ldw, (int)ldw, m, smem, smem_cap, ds);
    SID_MARK(18)
    if (pf) atomicAdd(reinterpret_cast<unsigned long long*>(sk.prof + 23), 1ull);
    return ds != nullptr;
  }
  const int64_t ldw = max(1, gather_chunks<false>(lv, sk, nc, s, 0, nch, nullptr, 1, 0, sint, 512));
  SID_MARK(16)
  const bool local = ldw * k + 4 * (int64_t)k + 4 <= smem_cap;
  double* W = local ? smem + SMEM_DOUBLES : sk.work + sk.work_off[s];
  double* vn1 = W + (int64_t)k * ldw;
  double* vn2 = vn1 + k;
  int* iw = local ? reinterpret_cast<int*>(vn2 + k) : sk.iwork + sk.iwork_off[s];
  int* perm = iw;
  int* sidx = iw + k;
  int* flag = iw + 2 * k;
  int m;
  if (nch <= 512) {
    // the count pass left every chunk's keep mask and row prefix in sint: copy without
    // recomputing them (nothing has written sint since)
    const unsigned* smask = reinterpret_cast<const unsigned*>(sint);
    const int* spre = sint + 512;
    const int g0 = sk.groups[s], warp = tid >> 5;
    for (int j = warp; j < nch; j += NT / 32) {
      const int i = nc.locate(j);
      chunk_copy<8>(lv, nc, g0, k, i, 32 * (j - nc.ch0[i]), smask[j], W, ldw, spre[j]);
    }
    m = nch > 0 ? spre[nch - 1] + __popc(smask[nch - 1]) : 0;
    __syncthreads();
  } else {
    m = gather_chunks<true>(lv, sk, nc, s, 0, nch, W, ldw, 0, sint, 512);
  }
  if (tid == 0) sk.rows[s] = m;
  SID_MARK(17)
  uint8_t* red = sk.red + gof;
  if (m == 0) {
    skel_all_redundant(lv, sk, s);
    return false;
  }
  if (sk.gram) {
    __syncthreads();   // gathered rows visible to every warp
    if (skel_id_gram(lv, sk, s, k, W, ldw, m, m, smem, smem_cap, ds)) {
      SID_MARK(18)
      if (pf) atomicAdd(reinterpret_cast<unsigned long long*>(sk.prof + 23), 1ull);
      return ds != nullptr;
    }
  }
#undef SID_MARK
  const double cutrel = fmax(sk.eps, DBL_EPSILON * (double)max(m, k));
  const int steps = cta_cpqr(W, m, k, ldw, perm, vn1, vn2, sred, cutrel);
  __shared__ int s_rank;
  if (tid == 0) {
    const double cut = cutrel * fabs(W[0]);
    int r = 0;
    for (int i = 0; i < steps; ++i)
      if (fabs(W[(int64_t)i * ldw + i]) > cut) ++r;
    s_rank = r;
    for (int j = 0; j < k; ++j) flag[j] = 0;
    for (int i = r; i < k; ++i) flag[perm[i]] = 1;
    int ns = 0, nr = 0;
    for (int j = 0; j < k; ++j) sidx[j] = flag[j] ? nr++ : ns++;
  }
  __syncthreads();
  const int r = s_rank, kt = k - r;
  // T = R11^-1 R12 (pivot order), in place over R12 columns
  for (int j = r + tid; j < k; j += NT) {
    double* cj = W + (int64_t)j * ldw;
    for (int i = r - 1; i >= 0; --i) {
      double v = cj[i];
      for (int l = i + 1; l < r; ++l) v -= W[(int64_t)l * ldw + i] * cj[l];
      cj[i] = v / W[(int64_t)i * ldw + i];
    }
  }
  __syncthreads();
  double* T = sk.rec + sk.T_off[s];
  for (int64_t e = tid; e < (int64_t)r * kt; e += NT) {
    const int i = (int)(e / kt), j = r + (int)(e % kt);
    T[(int64_t)sidx[perm[i]] * kt + sidx[perm[j]]] = W[(int64_t)j * ldw + i];
  }
  for (int j = tid; j < k; j += NT) {
    red[j] = (uint8_t)flag[j];
    if (flag[j]) sk.alive[lv.mem[gof + j]] = 0;
  }
  if (tid == 0) sk.rank[s] = r;
  return false;
}

__global__ void __launch_bounds__(NT) k_skel_id(LevelDev lv, SkelArgs sk, int smem_cap) {
  __shared__ NbrCache nc;
  const int s = sk.order[blockIdx.x];
  const bool pre = skel_id_pre(lv, sk, s, smem_cap, nc);
  skel_id_one(lv, sk, s, smem_cap, nc, pre, nullptr);
}

// Persistent, dependency-driven separator IDs (no wave barriers): CTAs take separators in a
// topological order (the wave order) from a counter, wait until every earlier coupled separator
// is done, run the ID, then release the later coupled ones. All CTAs are resident, and each
// waits only for items handed out before its own, so the chain always makes progress.
// MINB = 3 (80 registers, a few spilled) for levels of tiny separators (k <= 12: occupancy wins,
// level-0 ID of c5 7.3 -> 5.6 ms); MINB = 2 keeps the pivot-chain state of larger ones in registers.
template <int MINB>
__global__ void __launch_bounds__(NT, MINB) k_skel_id_dyn(LevelDev lv, SkelArgs sk, int smem_cap, DynSched ds) {
  __shared__ int s_item;
  __shared__ NbrCache nc;
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(ds.next, 1);
    __syncthreads();
    const int q = s_item;
    if (q >= ds.count) break;
    const int s = sk.order[q];
    // everything that does not depend on the earlier separators first (metadata, row staging)
    const bool pre = skel_id_pre(lv, sk, s, smem_cap, nc);
    const long long tw0 = (sk.prof && blockIdx.x == 0 && threadIdx.x == 0) ? clock64() : 0;
    if (threadIdx.x == 0) {
      volatile int* d = ds.done + s;
      const int nd = ds.ndep[s];
      while (*d < nd) __nanosleep(64);
      __threadfence();
    }
    __syncthreads();
    if (sk.prof && blockIdx.x == 0 && threadIdx.x == 0)
      atomicAdd(reinterpret_cast<unsigned long long*>(sk.prof + 19), (unsigned long long)(clock64() - tw0));
    const bool released = skel_id_one(lv, sk, s, smem_cap, nc, pre, &ds);
    __syncthreads();
    if (threadIdx.x == 0 && !released) {
      __threadfence();
      for (int64_t e = ds.succ_off[s]; e < ds.succ_off[s + 1]; ++e) atomicAdd(ds.done + ds.succ[e], 1);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Team CPQR: one separator per team of P co-resident CTAs (cooperative launch).
// Column j is owned by CTA j % P; per pivot step two team barriers: after the
// local argmax, and after the owner of column i swapped in the pivot and formed
// the reflector. Same arithmetic as cta_cpqr (dlaqp2 semantics).
// All loads of data written by other CTAs bypass L1 (ld.global.cg).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void team_sync(TeamHdr* h, int P) {
  __syncthreads();
  if (threadIdx.x == 0 && P > 1) {
    volatile unsigned* vgen = &h->gen;
    const unsigned g0 = *vgen;
    __threadfence();
    if (atomicAdd(&h->count, 1u) == (unsigned)(P - 1)) {
      h->count = 0;
      __threadfence();
      atomicAdd(&h->gen, 1u);
    } else {
      while (*vgen == g0) __nanosleep(40);
    }
    __threadfence();
  }
  __syncthreads();
}

// team barrier: a hardware cluster barrier when the team is a thread-block cluster, else the
// global-memory barrier above (cooperative launch)
__device__ __forceinline__ void tsync(TeamHdr* h, int P, bool cl) {
  if (cl) {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  } else {
    team_sync(h, P);
  }
}

constexpr int TCH = 16;      // owned columns updated together per pass

// Copy jb (<= 8) columns of n rows between a global column block (ld gld, L1 bypassed: the
// data is written by other CTAs of the team) and a packed shared-memory panel (ld n).
// Loads of all columns are issued before any is consumed (16 in flight per thread).
// VMASK: rows above the diagonal read as 0 and the diagonal as 1 (unit reflectors V).
template <bool VMASK>
__device__ __forceinline__ void panel_load(double* dst, const double* src, int64_t gld, int jb, int n) {
  for (int r0 = 0; r0 < n; r0 += 2 * NT) {
    double v[8][2];
#pragma unroll
    for (int jj = 0; jj < 8; ++jj)
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int rr = r0 + u * NT + threadIdx.x;
        double x = 0.0;
        if (jj < jb && rr < n) {
          if (!VMASK || rr > jj) x = __ldcg(src + (int64_t)jj * gld + rr);
          else if (rr == jj) x = 1.0;
        }
        v[jj][u] = x;
      }
#pragma unroll
    for (int jj = 0; jj < 8; ++jj)
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int rr = r0 + u * NT + threadIdx.x;
        if (jj < jb && rr < n) dst[(int64_t)jj * n + rr] = v[jj][u];
      }
  }
}
__device__ __forceinline__ void panel_store(double* dst, int64_t gld, const double* src, int jb, int n) {
  for (int jj = 0; jj < jb; ++jj)
    for (int rr = threadIdx.x; rr < n; rr += NT) __stcg(dst + (int64_t)jj * gld + rr, src[(int64_t)jj * n + rr]);
}

__device__ __forceinline__ int nloc_all(int k, int c, int P) { return c < k ? (k - c + P - 1) / P : 0; }
constexpr int TOWN = 512;    // max owned columns per CTA (smem norms)

// Team CPQR (dgeqp3/dlaqp2 semantics) of one large separator by a team of P co-resident CTAs.
//  * Column j is owned by CTA j % P; LAPACK's column interchanges are replayed on a replicated
//    logical permutation (inv: logical -> physical, pos: physical -> logical), so pivot ties
//    break on the same logical index as idamax and no data moves.
//  * The first `ns` owned columns of a CTA live in its shared memory (master copy, no per-step
//    L2 traffic); the rest are streamed from L2. Each CTA publishes its local pivot candidate
//    to a global staging column before the (single) team barrier of a step, so every CTA can
//    form the winning Householder reflector right after it.
//  * Only R's diagonal and strictly-upper part are kept (Q is never needed); the loop stops
//    once the largest remaining partial norm is below the rank cut (see cta_cpqr).
__global__ void __launch_bounds__(NT, 1) k_skel_team(LevelDev lv, SkelArgs sk, TeamArgs ta) {
  extern __shared__ double smem[];
  double* sred = smem + RED_OFF;
  double* sdot = smem + GEMM_OFF;               // [nw][TCH] partial dots, then [TCH] products
  double* vs = smem + SMEM_DOUBLES;             // reflector (rows > i), vcap doubles
  __shared__ double ovn1[TOWN], ovn2[TOWN];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = NT / 32;
  const long long t_kernel0 = clock64();
  const bool clmode = ta.cluster > 0;
  int f = 0;
  if (clmode) {
    f = blockIdx.x / ta.cluster;
  } else {
    while (f + 1 < ta.nface && ta.team_off[f + 1] <= (int)blockIdx.x) ++f;
  }
  const int c = blockIdx.x - ta.team_off[f];
  const int P = ta.team_off[f + 1] - ta.team_off[f];
  TeamHdr* hdr = ta.hdr + f;
  double* slot_v = ta.slot_v + 2 * ta.team_off[f];
  int* slot_i = ta.slot_i + 2 * ta.team_off[f];
  double* cand_base = ta.cand + (int64_t)2 * ta.team_off[f] * ta.cand_ld;   // 2P staging columns
  const int s = ta.face[f];
  const int g = sk.groups[s];
  const int k = lv.gsize[g];
  const int64_t gof = lv.goff[g];
  __shared__ NbrCache nc;
  nbr_cache_load(lv, sk, s, nc);
  const int64_t ldw = nc.rows;
  double* W = sk.work + sk.work_off[s];
  int* iw = sk.iwork + sk.iwork_off[s];
  int* perm = iw;
  int* sidx = iw + k;
  int* flag = iw + 2 * k;
  int* inv = reinterpret_cast<int*>(vs + ta.vcap);   // k ints
  int* pos = inv + k;                                // k ints
  double* colbuf = vs + ta.vcap + k + 1;             // smem-resident owned columns (ld m)
  // ---- gather A_{R,I} across the team: CTA c takes a contiguous range of 32-row chunks; a
  //      team-wide prefix over the per-CTA kept counts places its rows (neighbour order kept)
  int m0;
  {
    int* sint = reinterpret_cast<int*>(smem + GEMM_OFF);
    const int nch = nc.nch;
    const int per = (nch + P - 1) / P;
    const int ch_lo = min(nch, c * per), ch_hi = min(nch, ch_lo + per);
    const int mine = gather_chunks<false>(lv, sk, nc, s, ch_lo, ch_hi, W, ldw, 0, sint, 512);
    if (tid == 0) __stcg(slot_i + c, mine);
    tsync(hdr, P, clmode);
    int before = 0, all = 0;
    for (int q2 = 0; q2 < P; ++q2) {
      const int v = __ldcg(slot_i + q2);
      if (q2 < c) before += v;
      all += v;
    }
    m0 = all;
    gather_chunks<true>(lv, sk, nc, s, ch_lo, ch_hi, W, ldw, before, sint, 512);
    if (c == 0 && tid == 0) sk.rows[s] = m0;
    tsync(hdr, P, clmode);
  }
  if (m0 == 0) {
    if (c == 0) skel_all_redundant(lv, sk, s);
    return;
  }
  // ---- row reduction: blocked Householder QR W = Q [R0; 0] (m0 > k) -----------------------
  // CPQR pivots depend only on A^T A, so the CPQR of R0 selects the same columns as the CPQR
  // of A (up to rounding) while every later step touches k instead of m0 rows.
  // Panels of nbq columns; block b (its columns) is owned by CTA b % P. The owner of block
  // pi+1 applies panel pi to it first, factors it at once and publishes it (hdr->qr_done,
  // look-ahead); everyone else applies published panels to their blocks with DMMA
  // (X -= V T^T V^T X) and only waits for the panel it needs next. No team barriers.
  int m = m0;
  const long long t_qr0 = clock64();
  // shared memory free in this phase: everything (reductions and staging are static here)
  const int64_t qcap = (int64_t)SMEM_DOUBLES + ta.vcap + ta.kmax + 1 + ta.colcap;
  if (m0 > k && 2 * (int64_t)m0 <= qcap) {
    const int nbq = (int)(qcap / (2 * (int64_t)m0) < 8 ? qcap / (2 * (int64_t)m0) : 8);
    const int npan = (k + nbq - 1) / nbq;
    double* const vbuf0 = smem;
    double* const vbuf1 = smem + (int64_t)nbq * m0;
    __shared__ double s_T[2][64];
    __shared__ double s_par[20];
    __shared__ double s_red[8][8];
    __shared__ double s_Y[8][64];
    __shared__ double s_Z[64];
    double* qt = ta.qt + (int64_t)f * ta.qt_ld;
    const bool qprof = ta.prof && blockIdx.x == 0 && tid == 0;
    const int g8 = lane >> 2, t4 = lane & 3;
    // factor panel pi (already updated by panels < pi) in smem, write it back and publish it
    auto factor = [&](int pi, bool preloaded) {
      long long tq0 = qprof ? clock64() : 0;
      if (qprof) ta.prof[20] += 1;
      const int j0 = pi * nbq, jb = min(nbq, k - j0), ldp = m0 - j0;
      double* Pn = (pi & 1) ? vbuf1 : vbuf0;
      double* Ts = s_T[pi & 1];
      if (!preloaded) panel_load<false>(Pn, W + (int64_t)j0 * ldw + j0, ldw, jb, ldp);
      __syncthreads();
      long long tf = qprof ? clock64() : 0;
      auto flap = [&](int slot) {
        if (qprof) {
          const long long t1 = clock64();
          ta.prof[slot] += t1 - tf;
          tf = t1;
        }
      };
      if (qprof) ta.prof[22] += tf - tq0;
      constexpr int PQ = 10;   // panel rows per thread held in registers
      if (ldp <= PQ * NT) {
        // register-resident panel: thread tid holds rows tid + q*NT of all (<= 8) columns; the
        // column loop is unrolled so every register index is static. Row jj < 8 lives in thread jj.
        double pr[PQ][8];
#pragma unroll
        for (int q = 0; q < PQ; ++q) {
          const int rr = tid + q * NT;
#pragma unroll
          for (int u = 0; u < 8; ++u) pr[q][u] = (rr < ldp && u < jb) ? Pn[(int64_t)u * ldp + rr] : 0.0;
        }
        __shared__ double s_row[8];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          if (jj < jb) {
            if (tid == jj) {
#pragma unroll
              for (int u = 0; u < 8; ++u) s_row[u] = pr[0][u];
            }
            double acc[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) acc[u] = 0.0;
#pragma unroll
            for (int q = 0; q < PQ; ++q) {
              const int rr = tid + q * NT;
              if (rr > jj && rr < ldp) {
                const double x = pr[q][jj];
                acc[0] += x * x;
#pragma unroll
                for (int u = 1; jj + u < 8; ++u) acc[u] += x * pr[q][jj + u];
              }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const double t2 = warp_sum(acc[u]);
              if (lane == 0) s_red[warp][u] = t2;
            }
            __syncthreads();
            if (warp == 0) {
              double mys = 0.0;
              if (lane < 8) {
#pragma unroll
                for (int w2 = 0; w2 < 8; ++w2) mys += s_red[w2][lane];
              }
              double sum[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) sum[u] = __shfl_sync(0xffffffffu, mys, u);
              if (lane == 0) {
                const double alpha = s_row[jj], xnorm = sqrt(sum[0]);
                double tau = 0.0, beta = alpha, scal = 1.0;
                if (xnorm != 0.0) {
                  beta = -copysign(hypot(alpha, xnorm), alpha);
                  tau = (beta - alpha) / beta;
                  scal = 1.0 / (alpha - beta);
                }
                Ts[jj * 8 + jj] = tau;
                s_par[0] = scal;
                s_par[16] = beta;
                for (int u = 1; u < 8; ++u) {
                  const double tw = (jj + u < jb) ? tau * (s_row[jj + u] + scal * sum[u]) : 0.0;   // tau v^T a_u
                  s_par[u] = tw * scal;
                  s_par[8 + u] = tw;
                }
              }
            }
            __syncthreads();
            const double scal = s_par[0];
            double cu[8];
#pragma unroll
            for (int u = 1; u < 8; ++u) cu[u] = s_par[u];
#pragma unroll
            for (int q = 0; q < PQ; ++q) {
              const int rr = tid + q * NT;
              if (rr > jj && rr < ldp) {
                const double x = pr[q][jj];
#pragma unroll
                for (int u = 1; jj + u < 8; ++u) pr[q][jj + u] -= cu[u] * x;
                pr[q][jj] = x * scal;
              }
            }
            if (tid == jj) {
              pr[0][jj] = s_par[16];
#pragma unroll
              for (int u = 1; jj + u < 8; ++u) pr[0][jj + u] -= s_par[8 + u];
            }
          }
        }
#pragma unroll
        for (int q = 0; q < PQ; ++q) {
          const int rr = tid + q * NT;
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (rr < ldp && u < jb) Pn[(int64_t)u * ldp + rr] = pr[q][u];
        }
        __syncthreads();
      } else
      for (int jj = 0; jj < jb; ++jj) {
        // one reduction per column: |x|^2 and x . a_u (x = column jj below the diagonal)
        double acc[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] = 0.0;
        const double* xc = Pn + (int64_t)jj * ldp;
        for (int rr = jj + 1 + tid; rr < ldp; rr += NT) {
          const double x = xc[rr];
          acc[0] += x * x;
#pragma unroll
          for (int u = 1; u < 8; ++u)
            if (jj + u < jb) acc[u] += x * Pn[(int64_t)(jj + u) * ldp + rr];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const double t2 = warp_sum(acc[u]);
          if (lane == 0) s_red[warp][u] = t2;
        }
        __syncthreads();
        if (warp == 0) {
          double mys = 0.0;
          if (lane < 8) {
#pragma unroll
            for (int w2 = 0; w2 < 8; ++w2) mys += s_red[w2][lane];
          }
          double sum[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) sum[u] = __shfl_sync(0xffffffffu, mys, u);
          if (lane == 0) {
          const double alpha = xc[jj], xnorm = sqrt(sum[0]);
          double tau = 0.0, beta = alpha, scal = 1.0;
          if (xnorm != 0.0) {
            beta = -copysign(hypot(alpha, xnorm), alpha);
            tau = (beta - alpha) / beta;
            scal = 1.0 / (alpha - beta);
          }
          Pn[(int64_t)jj * ldp + jj] = beta;
          Ts[jj * 8 + jj] = tau;
          s_par[0] = scal;
          for (int u = 1; u < 8; ++u)
            if (jj + u < jb) {
              double* au = Pn + (int64_t)(jj + u) * ldp;
              const double tw = tau * (au[jj] + scal * sum[u]);   // tau * v^T a_u
              au[jj] -= tw;
              s_par[u] = tw * scal;                               // a_u -= tw * scal * x (rows > jj)
            }
          }
        }
        __syncthreads();
        const double scal = s_par[0];
        double cu[8];
#pragma unroll
        for (int u = 1; u < 8; ++u) cu[u] = (jj + u < jb) ? s_par[u] : 0.0;
        for (int rr = jj + 1 + tid; rr < ldp; rr += NT) {
          const double x = Pn[(int64_t)jj * ldp + rr];
#pragma unroll
          for (int u = 1; u < 8; ++u)
            if (jj + u < jb) Pn[(int64_t)(jj + u) * ldp + rr] -= cu[u] * x;
          Pn[(int64_t)jj * ldp + rr] = x * scal;
        }
        __syncthreads();
      }
      flap(23);
      // compact WY factor T (upper triangular): H_1 ... H_jb = I - V T V^T, from G = V^T V
      {
        double gp[28];
#pragma unroll
        for (int q = 0; q < 28; ++q) gp[q] = 0.0;
        for (int rr = 1 + tid; rr < ldp; rr += NT) {
          double va[8];
#pragma unroll
          for (int a = 0; a < 8; ++a)
            va[a] = (a < jb && rr >= a) ? (rr == a ? 1.0 : Pn[(int64_t)a * ldp + rr]) : 0.0;
          int q = 0;
#pragma unroll
          for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int b2 = a + 1; b2 < 8; ++b2) gp[q++] += va[a] * va[b2];
        }
#pragma unroll
        for (int q = 0; q < 28; ++q) {
          const double t2 = warp_sum(gp[q]);
          if (lane == 0) s_Y[warp][q] = t2;
        }
        __syncthreads();
        __shared__ double s_G[8][8];
        if (tid < 28) {
          double x = 0.0;
#pragma unroll
          for (int w2 = 0; w2 < 8; ++w2) x += s_Y[w2][tid];
          int a = 0, q = tid;
          while (q >= 7 - a) {
            q -= 7 - a;
            ++a;
          }
          s_G[a][a + 1 + q] = x;
        }
        __syncthreads();
        // T(0:i, i) = -tau_i T(0:i, 0:i) G(0:i, i), one column at a time; lane a holds row a
        if (warp == 0) {
          const int a = lane;
          double Trow[8];
#pragma unroll
          for (int b2 = 0; b2 < 8; ++b2) Trow[b2] = 0.0;
#pragma unroll
          for (int i2 = 0; i2 < 8; ++i2) {
            if (i2 >= jb) break;
            const double ti = Ts[i2 * 8 + i2];
            double x = 0.0;
#pragma unroll
            for (int b2 = 0; b2 < 8; ++b2)
              if (b2 >= a && b2 < i2) x += Trow[b2] * s_G[b2][i2];
            if (a < i2) Trow[i2] = -ti * x;
            else if (a == i2) Trow[i2] = ti;
          }
          if (a < 8) {
#pragma unroll
            for (int b2 = 0; b2 < 8; ++b2) {
              const double v = (a < jb && b2 < jb) ? Trow[b2] : 0.0;
              Ts[a * 8 + b2] = v;
              if (a < jb && b2 < jb) __stcg(qt + (int64_t)pi * nbq * nbq + a * nbq + b2, v);
            }
          }
        }
      }
      flap(24);
      panel_store(W + (int64_t)j0 * ldw + j0, ldw, Pn, jb, ldp);
      __syncthreads();
      flap(25);
      if (tid == 0 && P > 1) {
        __threadfence();
        atomicAdd(&hdr->qr_done, 1u);
      }
      // the smem copy becomes the unit-lower V of this panel
      for (int e = tid; e < jb * jb; e += NT) {
        const int jj = e / jb, rr = e % jb;
        if (rr <= jj) Pn[(int64_t)jj * ldp + rr] = rr == jj ? 1.0 : 0.0;
      }
      __syncthreads();
      if (qprof) ta.prof[14] += clock64() - tq0;
    };
    // X(:, block b) -= V (T^T (V^T X)) for panel pi (V in Vb, T in Ts), rows j0.. of the block.
    // Rows are split across warps in 8-row tiles; inside a tile the K order of V^T X is
    // permuted (k-step z takes rows 2t+z) so each lane's B fragments are exactly its C
    // fragments of the transposed update X^T -= Z^T V^T: the block slice stays in registers
    // (QR_TPW tiles per warp; all loads issued at once), only the excess is re-read.
    // Pnext (look-ahead block b = pi+1 of this CTA): rows below the next panel's diagonal go to
    // the next panel buffer in shared memory instead of global memory (factor() skips its load)
    auto update = [&](int pi, int b, const double* Vb, const double* Ts, double* Pnext) {
      constexpr int QR_TPW = 40;
      const int j0 = pi * nbq, jb = min(nbq, k - j0), ldp = m0 - j0;
      const int cb0 = b * nbq, ncol = min(nbq, k - cb0);
      const int ntile = (ldp + 7) >> 3;
      const int tpw = (ntile + nw - 1) / nw;
      const int t_lo = warp * tpw, t_hi = min(ntile, t_lo + tpw);
      const bool col_ok = g8 < ncol, va_ok = g8 < jb;
      double* Xc = W + (int64_t)(cb0 + min(g8, ncol - 1)) * ldw + j0;
      const double* Va = Vb + (int64_t)min(g8, jb - 1) * ldp;
      long long tp0 = qprof ? clock64() : 0;
      double xr[QR_TPW][2];
#pragma unroll
      for (int u = 0; u < QR_TPW; ++u) {
        const int rr = (t_lo + u) * 8 + 2 * t4;
        const bool ok = t_lo + u < t_hi && col_ok;
        xr[u][0] = (ok && rr < ldp) ? __ldcg(Xc + rr) : 0.0;
        xr[u][1] = (ok && rr + 1 < ldp) ? __ldcg(Xc + rr + 1) : 0.0;
      }
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int u = 0; u < QR_TPW; ++u) {
        const int rr = (t_lo + u) * 8 + 2 * t4;
        if (t_lo + u < t_hi) {
          const double a0 = (va_ok && rr < ldp) ? Va[rr] : 0.0;
          const double a1 = (va_ok && rr + 1 < ldp) ? Va[rr + 1] : 0.0;
          dmma(c0, c1, a0, xr[u][0]);
          dmma(c0, c1, a1, xr[u][1]);
        }
      }
      for (int tl = t_lo + QR_TPW; tl < t_hi; ++tl) {   // beyond the register slice
        const int rr = tl * 8 + 2 * t4;
        const double x0 = (col_ok && rr < ldp) ? __ldcg(Xc + rr) : 0.0;
        const double x1 = (col_ok && rr + 1 < ldp) ? __ldcg(Xc + rr + 1) : 0.0;
        dmma(c0, c1, (va_ok && rr < ldp) ? Va[rr] : 0.0, x0);
        dmma(c0, c1, (va_ok && rr + 1 < ldp) ? Va[rr + 1] : 0.0, x1);
      }
      s_Y[warp][g8 * 8 + 2 * t4] = c0;
      s_Y[warp][g8 * 8 + 2 * t4 + 1] = c1;
      __syncthreads();
      if (qprof) {
        const long long t1 = clock64();
        ta.prof[16] += 1;
        ta.prof[17] += t1 - tp0;
        tp0 = t1;
      }
      if (tid < 64) {
        const int bz = tid >> 3, col = tid & 7;
        double z = 0.0;
        for (int a = 0; a <= bz; ++a) {
          double y = 0.0;
          for (int w2 = 0; w2 < nw; ++w2) y += s_Y[w2][a * 8 + col];
          z += Ts[a * 8 + bz] * y;
        }
        s_Z[tid] = z;
      }
      __syncthreads();
      if (qprof) {
        const long long t1 = clock64();
        ta.prof[18] += t1 - tp0;
        tp0 = t1;
      }
      // X^T -= Z^T V^T: M = columns, N = rows of the tile, K = reflectors (two k-steps)
      const double za0 = -s_Z[t4 * 8 + g8], za1 = -s_Z[(t4 + 4) * 8 + g8];
      const double* V0 = Vb + (int64_t)min(t4, jb - 1) * ldp;
      const double* V1 = Vb + (int64_t)min(t4 + 4, jb - 1) * ldp;
      const bool b0_ok = t4 < jb, b1_ok = t4 + 4 < jb;
#pragma unroll
      for (int u = 0; u < QR_TPW; ++u) {
        if (t_lo + u < t_hi) {
          const int rv = (t_lo + u) * 8 + g8;
          const double vb0 = (b0_ok && rv < ldp) ? V0[rv] : 0.0;
          const double vb1 = (b1_ok && rv < ldp) ? V1[rv] : 0.0;
          dmma(xr[u][0], xr[u][1], za0, vb0);
          dmma(xr[u][0], xr[u][1], za1, vb1);
          const int rr = (t_lo + u) * 8 + 2 * t4;
          if (col_ok) {
            if (Pnext) {
              const int ldn = ldp - nbq;
              if (rr < ldp) {
                if (rr < nbq) __stcg(Xc + rr, xr[u][0]);
                else Pnext[(int64_t)g8 * ldn + rr - nbq] = xr[u][0];
              }
              if (rr + 1 < ldp) {
                if (rr + 1 < nbq) __stcg(Xc + rr + 1, xr[u][1]);
                else Pnext[(int64_t)g8 * ldn + rr + 1 - nbq] = xr[u][1];
              }
            } else {
              if (rr < ldp) __stcg(Xc + rr, xr[u][0]);
              if (rr + 1 < ldp) __stcg(Xc + rr + 1, xr[u][1]);
            }
          }
        }
      }
      for (int tl = t_lo + QR_TPW; tl < t_hi; ++tl) {
        const int rr = tl * 8 + 2 * t4, rv = tl * 8 + g8;
        double x0 = (col_ok && rr < ldp) ? __ldcg(Xc + rr) : 0.0;
        double x1 = (col_ok && rr + 1 < ldp) ? __ldcg(Xc + rr + 1) : 0.0;
        dmma(x0, x1, za0, (b0_ok && rv < ldp) ? V0[rv] : 0.0);
        dmma(x0, x1, za1, (b1_ok && rv < ldp) ? V1[rv] : 0.0);
        if (col_ok) {
          if (Pnext) {
            const int ldn = ldp - nbq;
            if (rr < ldp) {
              if (rr < nbq) __stcg(Xc + rr, x0);
              else Pnext[(int64_t)g8 * ldn + rr - nbq] = x0;
            }
            if (rr + 1 < ldp) {
              if (rr + 1 < nbq) __stcg(Xc + rr + 1, x1);
              else Pnext[(int64_t)g8 * ldn + rr + 1 - nbq] = x1;
            }
          } else {
            if (rr < ldp) __stcg(Xc + rr, x0);
            if (rr + 1 < ldp) __stcg(Xc + rr + 1, x1);
          }
        }
      }
      __syncthreads();
      if (qprof) ta.prof[19] += clock64() - tp0;
    };
    if (c == 0) factor(0, false);
    for (int pi = 0; pi < npan; ++pi) {
      double* Vb = (pi & 1) ? vbuf1 : vbuf0;
      const double* Ts = s_T[pi & 1];
      if (pi % P != c) {
        long long tq0 = qprof ? clock64() : 0;
        if (qprof) ta.prof[21] += 1;
        if (tid == 0) {
          volatile unsigned* done = &hdr->qr_done;
          while (*done < (unsigned)(pi + 1)) __nanosleep(32);
          __threadfence();
        }
        __syncthreads();
        if (qprof) {
          const long long t1 = clock64();
          ta.prof[15] += t1 - tq0;
          tq0 = t1;
        }
        const int j0 = pi * nbq, jb = min(nbq, k - j0);
        panel_load<true>(Vb, W + (int64_t)j0 * ldw + j0, ldw, jb, m0 - j0);
        if (tid < 64) {
          const int a = tid >> 3, b2 = tid & 7;
          s_T[pi & 1][tid] = (a < jb && b2 < jb) ? __ldcg(qt + (int64_t)pi * nbq * nbq + a * nbq + b2) : 0.0;
        }
        __syncthreads();
        if (qprof) ta.prof[7] += clock64() - tq0;
      }
      long long tu0 = qprof ? clock64() : 0;
      int b = pi + 1 + ((c - (pi + 1)) % P + P) % P;   // first owned block > pi
      if (b == pi + 1 && b < npan) {
        update(pi, b, Vb, Ts, ((pi + 1) & 1) ? vbuf1 : vbuf0);
        if (qprof) ta.prof[7] += clock64() - tu0;
        factor(b, true);
        tu0 = qprof ? clock64() : 0;
        b += P;
      }
      for (; b < npan; b += P) update(pi, b, Vb, Ts, nullptr);
      if (qprof) ta.prof[7] += clock64() - tu0;
    }
    tsync(hdr, P, clmode);
    // R0 = rows 0..k-1 of W: clear the reflector entries below the diagonal of owned columns
    for (int t = 0; t < nloc_all(k, c, P); ++t) {
      const int j = c + P * t;
      double* cj = W + (int64_t)j * ldw;
      for (int rr = j + 1 + tid; rr < k; rr += NT) __stcg(cj + rr, 0.0);
    }
    m = k;
    tsync(hdr, P, clmode);
  }
  if (ta.prof && blockIdx.x == 0 && tid == 0) ta.prof[11] += clock64() - t_qr0;
  const long long t_cp0 = clock64();
  const int nloc = nloc_all(k, c, P);                 // owned columns j = c + P*t
  const int ncap = ta.colcap / m;
  const int ns = min(nloc, ncap);                     // owned columns t < ns live in smem
  const bool v_in_smem = m <= ta.vcap;
  const double tol3z = sqrt(DBL_EPSILON * 0.5);
  for (int j = tid; j < k; j += NT) {
    inv[j] = j;
    pos[j] = j;
  }
  for (int t0 = 0; t0 < ns; t0 += 8)
    panel_load<false>(colbuf + (int64_t)t0 * m, W + (int64_t)(c + P * t0) * ldw, (int64_t)P * ldw, min(8, ns - t0), m);
  __syncthreads();
  for (int t = warp; t < nloc; t += nw) {
    double a = 0.0;
    if (t < ns) {
      const double* cj = colbuf + (int64_t)t * m;
      for (int r = lane; r < m; r += 32) a += cj[r] * cj[r];
    } else {
      const double* cj = W + (int64_t)(c + P * t) * ldw;
      for (int r = lane; r < m; r += 32) {
        const double x = __ldcg(cj + r);
        a += x * x;
      }
    }
    a = sqrt(warp_sum(a));
    if (lane == 0) ovn1[t] = ovn2[t] = a;
  }
  __syncthreads();
  const int mn = min(m, k);
  double* diagR = W + (int64_t)k * ldw;   // R_ii of completed steps
  const double cutrel = fmax(sk.eps, DBL_EPSILON * (double)max(m0, k));
  double cut = 0.0;
  int steps = 0;
  const bool prof = ta.prof && blockIdx.x == 0 && tid == 0;
  long long tp = prof ? clock64() : 0;
#define TEAM_PHASE(id)                                   \
  if (prof) {                                            \
    const long long now = clock64();                     \
    ta.prof[id] += now - tp;                             \
    tp = now;                                            \
  }
  for (int i = 0; i < mn; ++i) {
    // (a) local argmax over owned unpivoted columns: value, then logical position (idamax)
    ArgMax loc{-1.0, 0x7fffffff};
    for (int t = tid; t < nloc; t += NT) {
      const int pj = pos[c + P * t];
      if (pj >= i) loc = better(loc, ArgMax{ovn1[t], pj});
    }
    const ArgMax mine = cta_argmax(loc, sred);
    // publish the local candidate if it lives in shared memory
    if (mine.i != 0x7fffffff) {
      const int tb = (inv[mine.i] - c) / P;
      if (tb < ns) {
        const double* src = colbuf + (int64_t)tb * m;
        double* dst = cand_base + (int64_t)(((i & 1) * P) + c) * ta.cand_ld;
        for (int r = i + tid; r < m; r += NT) __stcg(dst + r, src[r]);
      }
    }
    const int par = (i & 1) * P;
    if (tid == 0) {
      __stcg(slot_v + par + c, mine.v);
      __stcg(slot_i + par + c, mine.i);
    }
    TEAM_PHASE(0);
    tsync(hdr, P, clmode);
    TEAM_PHASE(1);
    ArgMax cand{-1.0, 0x7fffffff};
    for (int q = tid; q < P; q += NT) cand = better(cand, ArgMax{__ldcg(slot_v + par + q), __ldcg(slot_i + par + q)});
    const ArgMax best = cta_argmax(cand, sred);
    // early exit: pivot norms do not increase, so once the largest remaining partial norm is
    // clearly below the rank cut no later |R_jj| can pass it; R11 and R12 are final already
    if (i > 0 && best.v < cut * (1.0 - 1e-4)) break;
    const int p = best.i;
    const int phys = inv[p];
    const int q = phys % P, tq = (phys - q) / P;
    const int nloc_q = q < k ? (k - q + P - 1) / P : 0;
    const double* cp = (tq < min(nloc_q, ncap)) ? cand_base + (int64_t)(((i & 1) * P) + q) * ta.cand_ld
                                                : W + (int64_t)phys * ldw;
    __syncthreads();
    if (tid == 0 && p != i) {   // replay the interchange on the logical permutation
      const int a = inv[i];
      inv[i] = phys;
      inv[p] = a;
      pos[a] = p;
      pos[phys] = i;
    }
    // (b) reflector of the pivot column (dlarfg), formed by every CTA
    double part = 0.0;
    for (int r = i + 1 + tid; r < m; r += NT) {
      const double x = __ldcg(cp + r);
      if (v_in_smem) vs[r] = x;
      part += x * x;
    }
    const double xnorm = sqrt(cta_sum(part, sred));   // cta_sum syncs: inv/pos/vs visible
    const double alpha = __ldcg(cp + i);
    double tau = 0.0, beta = alpha, scal = 1.0;
    if (xnorm != 0.0) {
      beta = -copysign(hypot(alpha, xnorm), alpha);
      tau = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    TEAM_PHASE(2);
    if (i == 0) cut = cutrel * fabs(beta);
    if (c == 0 && tid == 0) __stcg(diagR + i, beta);
    steps = i + 1;
    // (c) apply H = I - tau [1; v][1; v]^T (v = scal * x) to the owned unpivoted columns: one
    //     warp per column (dot, update and the dlaqp2 partial-norm downdate stay in the warp)
    for (int t = warp; t < nloc; t += nw) {
      if (pos[c + P * t] <= i) continue;
      const bool sm = t < ns;
      double* cj = sm ? colbuf + (int64_t)t * m : W + (int64_t)(c + P * t) * ldw;
      double rowi = sm ? cj[i] : __ldcg(cj + i);
      if (tau != 0.0) {
        double w = 0.0;
        for (int r = i + 1 + lane; r < m; r += 32) {
          const double vr = v_in_smem ? vs[r] : __ldcg(cp + r);
          w += vr * (sm ? cj[r] : __ldcg(cj + r));
        }
        w = warp_sum(w);
        const double tw = tau * (rowi + scal * w);
        rowi -= tw;
        const double tws = tw * scal;
        for (int r = i + 1 + lane; r < m; r += 32) {
          const double vr = v_in_smem ? vs[r] : __ldcg(cp + r);
          if (sm) cj[r] -= tws * vr;
          else __stcg(cj + r, __ldcg(cj + r) - tws * vr);
        }
        if (lane == 0) {
          if (sm) cj[i] = rowi;
          else __stcg(cj + i, rowi);
        }
      }
      // partial-norm downdate (dlaqp2 loop 10) on the updated pivot-row entry
      const double v1 = ovn1[t];
      bool rec = false;
      if (v1 != 0.0) {
        double tt = fabs(rowi) / v1;
        tt = 1.0 - tt * tt;
        tt = tt < 0.0 ? 0.0 : tt;
        const double rr = v1 / ovn2[t];
        if (tt * rr * rr <= tol3z) rec = true;
        else if (lane == 0) ovn1[t] = v1 * sqrt(tt);
      }
      if (rec) {
        __syncwarp();
        double a = 0.0;
        if (i < m - 1) {
          for (int r = i + 1 + lane; r < m; r += 32) {
            const double x = sm ? cj[r] : __ldcg(cj + r);
            a += x * x;
          }
          a = sqrt(warp_sum(a));
        }
        if (lane == 0) ovn1[t] = ovn2[t] = a;
      }
    }
    __syncthreads();
    TEAM_PHASE(5);
    if (prof) ta.prof[8] += 1;
  }
#undef TEAM_PHASE
  if (ta.prof && blockIdx.x == 0 && tid == 0) ta.prof[12] += clock64() - t_cp0;
  const long long t_fin0 = clock64();
  // write back R rows [0, steps) of shared-memory columns
  for (int64_t e = tid; e < (int64_t)ns * steps; e += NT) {
    const int t = (int)(e / steps), r = (int)(e % steps);
    __stcg(W + (int64_t)(c + P * t) * ldw + r, colbuf[(int64_t)t * m + r]);
  }
  tsync(hdr, P, clmode);
  // rank from the diagonal (identical on every CTA); natural-order maps by CTA 0
  __shared__ int s_rank;
  {
    const double cutv = cutrel * fabs(__ldcg(diagR));
    int cnt = 0;
    for (int i = tid; i < steps; i += NT) cnt += fabs(__ldcg(diagR + i)) > cutv ? 1 : 0;
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    __shared__ int s_cnt[NT / 32];
    if (lane == 0) s_cnt[warp] = cnt;
    __syncthreads();
    if (tid == 0) {
      int r = 0;
      for (int w2 = 0; w2 < nw; ++w2) r += s_cnt[w2];
      s_rank = r;
    }
    __syncthreads();
  }
  if (c == 0) {
    // redundant flags, permutation and the natural-order skeleton/redundant indices
    const int r = s_rank;
    for (int j = tid; j < k; j += NT) {
      __stcg(flag + j, 0);
      __stcg(perm + j, inv[j]);
    }
    __syncthreads();
    for (int i = r + tid; i < k; i += NT) __stcg(flag + inv[i], 1);
    __syncthreads();
    int* sint = reinterpret_cast<int*>(sred);
    int base_s = 0, base_r = 0;
    for (int j0 = 0; j0 < k; j0 += NT) {
      const int j = j0 + tid;
      const int fl = j < k ? __ldcg(flag + j) : 0;
      int tot;
      const int off = cta_scan_flag(fl, sint, &tot);
      if (j < k) __stcg(sidx + j, fl ? base_r + off : base_s + (tid - off));
      base_r += tot;
      base_s += min(NT, k - j0) - tot;
    }
  }
  tsync(hdr, P, clmode);
  const int r = s_rank, kt = k - r;
  // T = R11^-1 R12: owned physical columns at logical positions >= r (warp per column).
  // Column-oriented back substitution: the right-hand side stays in registers (lane holds rows
  // lane + 32q), x_l is broadcast by a shuffle and R11's column l (contiguous, not written in
  // this phase, so read through L1 and shared by the CTA's warps) updates the rows above l.
  constexpr int TQ = 16;
  for (int ph = c + P * warp; ph < k && r <= 32 * TQ; ph += P * nw) {
    if (pos[ph] < r) continue;
    double* cj = W + (int64_t)ph * ldw;
    double bq[TQ];
#pragma unroll
    for (int q = 0; q < TQ; ++q) bq[q] = lane + 32 * q < r ? __ldcg(cj + lane + 32 * q) : 0.0;
    for (int l = r - 1; l >= 0; --l) {
      const int ql = l >> 5, ll = l & 31;
      double bl = 0.0;
#pragma unroll
      for (int q = 0; q < TQ; ++q)
        if (q == ql) bl = bq[q];
      const double xl = __shfl_sync(0xffffffffu, bl, ll) / __ldcg(diagR + l);
      const double* Rl = W + (int64_t)inv[l] * ldw;
#pragma unroll
      for (int q = 0; q < TQ; ++q) {
        const int row = lane + 32 * q;
        if (row < l) bq[q] -= xl * __ldg(Rl + row);
        else if (row == l) bq[q] = xl;
      }
    }
#pragma unroll
    for (int q = 0; q < TQ; ++q)
      if (lane + 32 * q < r) __stcg(cj + lane + 32 * q, bq[q]);
  }
  for (int ph = c + P * warp; ph < k && r > 32 * TQ; ph += P * nw) {
    if (pos[ph] < r) continue;
    double* cj = W + (int64_t)ph * ldw;
    for (int l = r - 1; l >= 0; --l) {
      double a = 0.0;
      for (int l2 = l + 1 + lane; l2 < r; l2 += 32) a += __ldcg(W + (int64_t)inv[l2] * ldw + l) * __ldcg(cj + l2);
      a = warp_sum(a);
      __syncwarp();
      if (lane == 0) __stcg(cj + l, (__ldcg(cj + l) - a) / __ldcg(diagR + l));
      __syncwarp();
    }
  }
  __syncthreads();
  double* T = sk.rec + sk.T_off[s];
  for (int ph = c; ph < k; ph += P) {
    if (pos[ph] < r) continue;
    const int col = __ldcg(sidx + ph);
    for (int l = tid; l < r; l += NT) T[(int64_t)__ldcg(sidx + inv[l]) * kt + col] = __ldcg(W + (int64_t)ph * ldw + l);
  }
  if (ta.prof && tid == 0) atomicAdd((unsigned long long*)&ta.prof[9 + (c == 0 ? 0 : 1)], (unsigned long long)(clock64() - t_kernel0));
  if (ta.prof && blockIdx.x == 0 && tid == 0) ta.prof[13] += clock64() - t_fin0;
  if (c == 0) {
    uint8_t* red = sk.red + gof;
    for (int j = tid; j < k; j += NT) {
      const int fl = __ldcg(flag + j);
      red[j] = (uint8_t)fl;
      if (fl) sk.alive[lv.mem[gof + j]] = 0;
    }
    if (tid == 0) sk.rank[s] = r;
  }
}

// ---------------------------------------------------------------------------
// Stage 3b: zeroing + elimination of the redundant DOFs.
// Panel [A~_rr ; A~_sr] ((kt+r) x kt) -> [L~ ; X~^T];  A_ss -= X~^T X~.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(NT, 3) k_skel_update(LevelDev lv, SkelArgs sk, const int* list, DevStatus* st) {
  extern __shared__ double smem[];
  const int tid = threadIdx.x;
  const int s = list ? list[blockIdx.x] : blockIdx.x;
  const int g = sk.groups[s];
  const int k = lv.gsize[g];
  const int r = sk.rank[s], kt = k - r;
  if (kt == 0) return;
  const uint8_t* red = sk.red + lv.goff[g];
  int* iw = sk.iwork + sk.iwork_off[s];
  int* skl = iw;       // r
  int* rdl = iw + k;   // kt
  if (tid == 0) {
    int a = 0, c = 0;
    for (int j = 0; j < k; ++j) {
      if (red[j]) rdl[c++] = j;
      else skl[a++] = j;
    }
  }
  __syncthreads();
  double* A = lv.pool + lv.boff[lv.diag_blk[g]];
  double* Pn = sk.rec + sk.P_off[s];
  const double* T = sk.rec + sk.T_off[s];
  double* Ass = sk.work + sk.work_off[s];
  double* Asr = Ass + (int64_t)r * r;
  for (int64_t e = tid; e < (int64_t)kt * kt; e += NT) {
    const int c = (int)(e / kt), d = (int)(e % kt);
    Pn[e] = A[(int64_t)rdl[c] * k + rdl[d]];
  }
  for (int64_t e = tid; e < (int64_t)r * r; e += NT) {
    const int a = (int)(e / r), b = (int)(e % r);
    Ass[e] = A[(int64_t)skl[a] * k + skl[b]];
  }
  double* Ast = Pn + (int64_t)kt * kt;
  for (int64_t e = tid; e < (int64_t)r * kt; e += NT) {
    const int a = (int)(e / kt), c = (int)(e % kt);
    const double v = A[(int64_t)skl[a] * k + rdl[c]];
    Asr[e] = v;
    Ast[e] = v;
  }
  double* Idr = Pn + (int64_t)(kt + r) * kt;   // identity rows: become L~^-T
  for (int64_t e = tid; e < (int64_t)kt * kt; e += NT) Idr[e] = (e / kt == e % kt) ? 1.0 : 0.0;
  __syncthreads();
  double* gsm = smem + GEMM_OFF;
  if (r > 0) {
    cta_gemm<false, false>(r, kt, r, -1.0, Ass, r, T, kt, 1.0, Ast, kt, false, gsm);      // Ast = Asr - Ass T
    cta_gemm<true, false>(kt, kt, r, -1.0, T, kt, Ast, kt, 1.0, Pn, kt, false, gsm);      // Att -= T^T Ast
    cta_gemm<true, false>(kt, kt, r, -1.0, Asr, kt, T, kt, 1.0, Pn, kt, false, gsm);      // Att -= Asr^T T
  }
  const int info = cta_potrf_panel(Pn, kt + r + kt, kt, kt, smem);
  if (info >= 0) {
    if (tid == 0) report_bad(st, s, info);
    return;
  }
  if (r > 0) {
    cta_gemm<false, true>(r, r, kt, -1.0, Ast, kt, Ast, kt, 1.0, Ass, r, false, gsm);     // A_ss -= X~^T X~
    for (int64_t e = tid; e < (int64_t)r * r; e += NT) {
      const int a = (int)(e / r), b = (int)(e % r);
      A[(int64_t)skl[a] * k + skl[b]] = Ass[e];
    }
  }
}

// Large separators (tile-parallel path): gather [A~_tt ; A~_st ; I] into the record and the
// work copies A_ss, A_sr (grid-stride over (separator, chunk)); skl/rdl = skeleton and
// redundant member positions per separator (host-built). The GEMMs, the panel Cholesky and
// U = X~^T X~ run as batched tile kernels; k_skel_big_post does A_ss -= U.
__global__ void k_skel_big_gather(LevelDev lv, SkelArgs sk, const int* big, const int* idx, const int64_t* idx_off,
                                  int nbig, int chunks) {
  const int bc = blockIdx.x / chunks, ch = blockIdx.x % chunks;
  if (bc >= nbig) return;
  const int s = big[bc];
  const int g = sk.groups[s], k = lv.gsize[g];
  const int r = sk.rank[s], kt = k - r;
  const int* skl = idx + idx_off[bc];
  const int* rdl = skl + r;
  const double* A = lv.pool + lv.boff[lv.diag_blk[g]];
  double* Pn = sk.rec + sk.P_off[s];
  double* Ast = Pn + (int64_t)kt * kt;
  double* Idr = Ast + (int64_t)r * kt;
  double* Ass = sk.work + sk.work_off[s];
  double* Asr = Ass + (int64_t)r * r;
  const int64_t stride = (int64_t)chunks * blockDim.x;
  const int64_t e0 = (int64_t)ch * blockDim.x + threadIdx.x;
  for (int64_t e = e0; e < (int64_t)kt * kt; e += stride) {
    const int a = (int)(e / kt), b = (int)(e % kt);
    Pn[e] = A[(int64_t)rdl[a] * k + rdl[b]];
    Idr[e] = a == b ? 1.0 : 0.0;
  }
  for (int64_t e = e0; e < (int64_t)r * r; e += stride) Ass[e] = A[(int64_t)skl[e / r] * k + skl[e % r]];
  for (int64_t e = e0; e < (int64_t)r * kt; e += stride) {
    const double v = A[(int64_t)skl[e / kt] * k + rdl[e % kt]];
    Asr[e] = v;
    Ast[e] = v;
  }
}
__global__ void k_skel_big_post(LevelDev lv, SkelArgs sk, const int* big, const int* idx, const int64_t* idx_off,
                                const double* U, const int64_t* U_off, int nbig, int chunks) {
  const int bc = blockIdx.x / chunks, ch = blockIdx.x % chunks;
  if (bc >= nbig) return;
  const int s = big[bc];
  const int g = sk.groups[s], k = lv.gsize[g];
  const int r = sk.rank[s];
  const int* skl = idx + idx_off[bc];
  double* A = lv.pool + lv.boff[lv.diag_blk[g]];
  const double* Ass = sk.work + sk.work_off[s];
  const double* Ub = U + U_off[bc];
  const int64_t stride = (int64_t)chunks * blockDim.x;
  for (int64_t e = (int64_t)ch * blockDim.x + threadIdx.x; e < (int64_t)r * r; e += stride)
    A[(int64_t)skl[e / r] * k + skl[e % r]] = Ass[e] - Ub[e];
}

// ---------------------------------------------------------------------------
// Big cells: 64-wide right-looking steps, every step tile-parallel over all
// big cells of the level (diag factor -> panel TRSM as GEMM with the explicit
// 64x64 inverse -> trailing update tiles), then U = X^T X by tiles.
// ---------------------------------------------------------------------------
constexpr int BT = 64, BLD = 65;

// one CTA per big cell still active at this step
__global__ void __launch_bounds__(NT) k_big_diag(BigArgs a, DevStatus* st) {
  // 64 x 64 Cholesky and triangular inverse. The trailing block lives in registers: warp w owns
  // rows w, w+8, ..., lane l owns columns l and l+32 (16 entries per thread). Each step publishes
  // one column (factor) or one row (inverse) in shared memory, double-buffered: one barrier per
  // step. The finished columns of L go to shared memory (Ls), from where the inverse reads its
  // multipliers as warp-wide broadcasts (issued before the step's barrier).
  __shared__ double colbuf[2][BT];
  __shared__ double dinv[BT];
  __shared__ double Ls[BT * BLD];
  __shared__ int sflag;
  const int c = a.w_cell[blockIdx.x];
  const int n = a.n[c], k0 = a.k0, kb = min(BT, n - k0);
  double* P = a.P[c];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  double Dr[8][2];
#pragma unroll
  for (int ri = 0; ri < 8; ++ri)
#pragma unroll
    for (int ci = 0; ci < 2; ++ci) {
      const int i = w + 8 * ri, cc = lane + 32 * ci;
      Dr[ri][ci] = (i < kb && cc <= i) ? P[(int64_t)(k0 + i) * n + k0 + cc] : (i == cc ? 1.0 : 0.0);
    }
  if (tid == 0) sflag = -1;
  for (int j = 0; j < BT; ++j) {
    const int par = j & 1, cj = j >> 5, lj = j & 31;
    if (lane == lj)
#pragma unroll
      for (int ri = 0; ri < 8; ++ri) {
        const int i = w + 8 * ri;
        if (i >= j) colbuf[par][i] = cj ? Dr[ri][1] : Dr[ri][0];   // (selects keep Dr in registers)
      }
    __syncthreads();
    const double djj = colbuf[par][j];
    if (!(djj > 0.0)) {
      if (tid == 0) sflag = j;
      break;
    }
    const double ljj = sqrt(djj), rj = 1.0 / ljj;
    // (column slot 0 holds columns <= 31: nothing left to update there once j >= 31)
    const double lc0 = (cj == 0 && lane > j) ? colbuf[par][lane] * rj : 0.0;
    const double lc1 = (lane + 32 > j) ? colbuf[par][lane + 32] * rj : 0.0;
#pragma unroll
    for (int ri = 0; ri < 8; ++ri) {
      const int i = w + 8 * ri;
      if (i > j) {
        const double li = colbuf[par][i] * rj;
        if (cj == 0 && lane > j && lane <= i) Dr[ri][0] = __fma_rn(-li, lc0, Dr[ri][0]);
        if (lane + 32 > j && lane + 32 <= i) Dr[ri][1] = __fma_rn(-li, lc1, Dr[ri][1]);
        if (lane == 0) Ls[i * BLD + j] = li;
      } else if (i == j) {
        if (lane == 0) Ls[i * BLD + j] = ljj;
      }
    }
    if (tid == 0) dinv[j] = rj;
  }
  __syncthreads();
  if (sflag >= 0) {
    if (tid == 0 && sflag < kb) report_bad(st, a.op[c], k0 + sflag);
    return;
  }
  // X = L^-1, right-looking: row j of X is final after scaling by 1/L(j,j); rows i > j then
  // subtract L(i,j) X(j,:). X(j, c) = 0 for c > j, so column slot 1 only takes part from j = 32.
  double Xr[8][2];
#pragma unroll
  for (int ri = 0; ri < 8; ++ri)
#pragma unroll
    for (int ci = 0; ci < 2; ++ci) Xr[ri][ci] = (w + 8 * ri == lane + 32 * ci) ? 1.0 : 0.0;
  for (int j = 0; j < BT; ++j) {
    const int par = j & 1, rj_i = j >> 3, wj = j & 7;
    double lij[8];
#pragma unroll
    for (int ri = 0; ri < 8; ++ri) lij[ri] = Ls[(w + 8 * ri) * BLD + j];   // (rows <= j: never used)
    if (w == wj) {
#pragma unroll
      for (int ri = 0; ri < 8; ++ri)
        if (ri == rj_i)
#pragma unroll
          for (int ci = 0; ci < 2; ++ci) {
            Xr[ri][ci] *= dinv[j];
            colbuf[par][lane + 32 * ci] = Xr[ri][ci];
          }
    }
    __syncthreads();
    const double x0 = colbuf[par][lane];
    if (j < 32) {
#pragma unroll
      for (int ri = 0; ri < 8; ++ri)
        if (w + 8 * ri > j) Xr[ri][0] = __fma_rn(-lij[ri], x0, Xr[ri][0]);
    } else {
      const double x1 = colbuf[par][lane + 32];
#pragma unroll
      for (int ri = 0; ri < 8; ++ri)
        if (w + 8 * ri > j) {
          Xr[ri][0] = __fma_rn(-lij[ri], x0, Xr[ri][0]);
          Xr[ri][1] = __fma_rn(-lij[ri], x1, Xr[ri][1]);
        }
    }
  }
  double* Lo = a.Linv + (int64_t)c * BT * BT;
#pragma unroll
  for (int ri = 0; ri < 8; ++ri)
#pragma unroll
    for (int ci = 0; ci < 2; ++ci) {
      const int i = w + 8 * ri, cc = lane + 32 * ci;
      Lo[i * BT + cc] = Xr[ri][ci];
      if (i < kb && cc < kb) P[(int64_t)(k0 + i) * n + k0 + cc] = (cc <= i) ? Ls[i * BLD + cc] : 0.0;
    }
  // (the strict upper part of the square block is zeroed once at the end: k_big_zero_upper)
}

// zero the strict upper triangle of every big panel's square part (never read by the steps)
__global__ void k_big_zero_upper(BigArgs a, int chunks) {
  const int c = blockIdx.x / chunks, ch = blockIdx.x % chunks;
  if (c >= a.ncell) return;
  const int n = a.n[c];
  double* P = a.P[c];
  for (int r = ch; r < n - 1; r += chunks)
    for (int j = r + 1 + (int)threadIdx.x; j < n; j += blockDim.x) P[(int64_t)r * n + j] = 0.0;
}

// acc += A (64 x 64) * B^T (64 x 64) on DMMA, both tiles row-major in smem, row stride TLD = 68
// (TLD mod 16 == 4: the 16 lanes of a half-warp, rows g < 4 and k offsets t < 4, read 16 different
// 8-byte banks; the stride 65 of the diagonal kernel gave 4-way conflicts on these fragments)
constexpr int TLD = 68;
__device__ __forceinline__ void tile_mma_nt(const double* sA, const double* sB, double acc[2][4][2]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp & 3, wn = warp >> 2, g = lane >> 2, t = lane & 3;
#pragma unroll 4
  for (int ks = 0; ks < BT; ks += 4) {
    double af[2], bf[4];
#pragma unroll
    for (int x = 0; x < 2; ++x) af[x] = sA[(wm * 16 + x * 8 + g) * TLD + ks + t];
#pragma unroll
    for (int y = 0; y < 4; ++y) bf[y] = sB[(wn * 32 + y * 8 + g) * TLD + ks + t];
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) dmma(acc[x][y][0], acc[x][y][1], af[x], bf[y]);
  }
}

__device__ __forceinline__ void cp_async8(void* smem_ptr, const void* gptr, bool pred);
__device__ __forceinline__ void cp_async_commit();
template <int N>
__device__ __forceinline__ void cp_async_wait();
// panel rows below the diagonal block: X = P[rows, k0:k0+64] * Linv^T (in place)
__global__ void __launch_bounds__(NT) k_big_trsm(BigArgs a) {
  extern __shared__ double smem[];
  double* sA = smem;
  double* sB = smem + BT * TLD;
  const int c = a.w_cell[blockIdx.x], it = a.w_i[blockIdx.x];
  const int n = a.n[c], rows = a.rows[c], k0 = a.k0, kb = min(BT, n - k0);
  const int r0 = k0 + kb + BT * it;
  double* P = a.P[c];
  const double* Li = a.Linv + (int64_t)c * BT * BT;
  const int tid = threadIdx.x;
  // both tiles by cp.async: the 32 copies of a thread are all in flight together (the plain
  // load -> store loop exposed the global latency several times per CTA)
#pragma unroll 4
  for (int e = tid; e < BT * BT; e += NT) {
    const int i = e / BT, j = e % BT;
    const bool ok = r0 + i < rows && j < kb;
    cp_async8(sA + i * TLD + j, P + (ok ? (int64_t)(r0 + i) * n + k0 + j : 0), ok);   // (zero fill)
    cp_async8(sB + i * TLD + j, Li + e, true);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  double acc[2][4][2] = {};
  tile_mma_nt(sA, sB, acc);
  const int lane = tid & 31, warp = tid >> 5, wm = warp & 3, wn = warp >> 2, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int z = 0; z < 2; ++z) {
        const int i = wm * 16 + x * 8 + g, j = wn * 32 + y * 8 + 2 * t + z;
        if (r0 + i < rows && j < kb) P[(int64_t)(r0 + i) * n + k0 + j] = acc[x][y][z];
      }
}

// build panels [A_gg ; I] of big block-Jacobi groups (A_gg <- I afterwards), grid-stride
__global__ void k_prec_build(LevelDev lv, PrecArgs pa, const int* list, int nbig, int chunks) {
  const int bc = blockIdx.x / chunks, ch = blockIdx.x % chunks;
  if (bc >= nbig) return;
  const int t = list[bc];
  const int g = pa.groups[t], k = lv.gsize[g];
  double* A = lv.pool + lv.boff[lv.diag_blk[g]];
  double* L = pa.rec + pa.L_off[t];
  const int64_t stride = (int64_t)chunks * blockDim.x;
  for (int64_t e = (int64_t)ch * blockDim.x + threadIdx.x; e < (int64_t)k * k; e += stride) {
    const double id = (e / k == e % k) ? 1.0 : 0.0;
    L[e] = A[e];
    L[(int64_t)k * k + e] = id;
    A[e] = id;
  }
}

// build panels [A_II ; A_BI] of big cells, grid-stride over (cell, chunk)
__global__ void k_big_build(LevelDev lv, CellArgs ca, const int* big_cells, int nbig, int chunks) {
  const int bc = blockIdx.x / chunks, ch = blockIdx.x % chunks;
  if (bc >= nbig) return;
  const int t = big_cells[bc];
  const int I = ca.interior[t], n = ca.n[t];
  double* P = ca.rec + ca.P_off[t];
  const double* A = lv.pool + lv.boff[lv.diag_blk[I]];
  const int64_t stride = (int64_t)chunks * blockDim.x;
  for (int64_t e = (int64_t)ch * blockDim.x + threadIdx.x; e < (int64_t)n * n; e += stride) P[e] = A[e];
  // A_BI rows: the block (I, h) is |I| x w row-major; its transpose lands in panel rows
  // n + c0 .. n + c0 + w. 32 x 32 tiles through shared memory (coalesced reads and writes).
  __shared__ double tile[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
  for (int64_t j = ca.nbr_off[t]; j < ca.nbr_off[t + 1]; ++j) {
    const int w = ca.nbr_w[j], c0 = ca.nbr_col[j];
    const double* S = lv.pool + lv.boff[ca.nbr_blk[j]];
    const int ti = (n + 31) / 32, tr = (w + 31) / 32;
    for (int tt = ch; tt < ti * tr; tt += chunks) {
      const int i0 = 32 * (tt / tr), r0 = 32 * (tt % tr);
      __syncthreads();
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + ty + 8 * u, r = r0 + tx;
        if (i < n && r < w) tile[ty + 8 * u][tx] = S[(int64_t)i * w + r];
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = r0 + ty + 8 * u, i = i0 + tx;
        if (i < n && r < w) P[(int64_t)(n + c0 + r) * n + i] = tile[tx][ty + 8 * u];
      }
    }
  }
  // identity rows below [A_II; A_BI]: the partial Cholesky turns them into L^-T (apply by GEMM)
  double* Id = P + (int64_t)(n + ca.b[t]) * n;
  for (int64_t e = (int64_t)ch * blockDim.x + threadIdx.x; e < (int64_t)n * n; e += stride)
    Id[e] = (e / n == e % n) ? 1.0 : 0.0;
}

// ---------------------------------------------------------------------------
// Batched skinny GEMM (replay of records, N = nrhs <= 32 per pass):
// C[64-row tile, 0:N] = beta*C + alpha*op(A)[rows, :] * B[:, 0:N].
// K is streamed in 32-wide chunks through a 2-stage cp.async pipeline; each warp
// owns 8 output rows x 32 columns (4 DMMA m8n8k4 tiles).
// ---------------------------------------------------------------------------
constexpr int SG_BM = 64, SG_BK = 32, SG_BN = 32;
constexpr int SG_ALD = SG_BK + 4;   // sA[row][k]   (A rows; +4 pad: conflict-free fragments)
constexpr int SG_BLD = SG_BN + 4;   // sB[k][col]
constexpr int SG_STAGE = SG_BM * SG_ALD + SG_BK * SG_BLD;

__device__ __forceinline__ void cp_async8(void* smem_ptr, const void* gptr, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_ptr);
  const int n = pred ? 8 : 0;   // src-size 0 -> zero fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gptr), "r"(n));
}
// 8-byte cp.async / read-only load with a 256-byte L2 prefetch: the records are streamed once in
// 256..512-byte row pieces, so every L2 miss fetches the whole piece from DRAM in one request
__device__ __forceinline__ void cp_async8_pf(void* smem_ptr, const void* gptr, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_ptr);
  const int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global.L2::256B [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gptr), "r"(n));
}
__device__ __forceinline__ double ldg_pf(const double* p) {
  double v;
  asm volatile("ld.global.nc.L2::256B.f64 %0, [%1];\n" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Replay GEMM for the factor apply (N = nrhs <= 32): C[64-row tile, 0:N] = beta*C + alpha*op(A) B.
// A (a stored record) is streamed once: each warp's m8n8k4 A fragments are read straight from
// global memory through the read-only path (8 full 32-byte sectors per load in either storage
// order); only the small right-hand-side chunk B[kc:kc+64, 0:N] is staged in shared memory.
// NT8 = ceil(N / 8) output column tiles per warp.
// The CTA walks its work items as one stream of 64-deep K chunks, pipelined ACROSS items: while
// chunk s is multiplied, the operands of chunk s+1 (possibly the first chunk of the next item)
// are in flight, and the descriptor of the item after that and the list entry of the one after
// that are prefetched. Records with K <= 64 (level-0/1 cells and separators) therefore cost one
// hidden round trip instead of four exposed ones. Arithmetic order per item is unchanged.
// RG_K = K depth of a chunk: 32 (3 CTAs per SM) for launches of shallow records, 64 (2 CTAs per SM,
// half the barriers and exposed steps) for deep ones; the host picks per launch from the mean K.
template <int NT8, int RG_K>
__global__ void __launch_bounds__(NT, RG_K == 32 ? 3 : 2) k_rgemm(const GemmDesc* __restrict__ desc, const int* __restrict__ w_desc,
                                                  const int* __restrict__ w_tile, int nwork, int N) {   // N = columns of every item (nrhs)
  constexpr int LDB = NT8 * 8 + 4;
  __shared__ double sB[2][RG_K * LDB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t4 = lane & 3;
  const int G = gridDim.x;
  // stage I: list entry (descriptor id, row tile) of the item three ahead
  int wI = blockIdx.x, pdI = -1, ptI = 0;
  auto fetchI = [&]() {
    pdI = -1;
    if (wI < nwork) {
      pdI = __ldg(w_desc + wI);
      ptI = __ldg(w_tile + wI);
    }
    wI += G;
  };
  // stage D: raw descriptor of the item two ahead
  const double *dA = nullptr, *dB = nullptr;
  int dM = 0, dK = 0, dlda = 0, dldb = 0, dtA = 0, dtri = 0, ddi = -1, di0 = 0;
  auto fetchD = [&]() {
    ddi = pdI;
    if (pdI >= 0) {
      const GemmDesc* p = desc + pdI;
      dA = p->A;
      dB = p->B;
      dM = p->M;
      dK = p->K;
      dlda = p->lda;
      dldb = p->ldb;
      dtA = p->transA;
      dtri = p->tri;
      di0 = 64 * ptI;
    }
    fetchI();
  };
  // stage L: the item whose chunks are being issued
  const double *lAr = nullptr, *lB = nullptr;
  int64_t lsk = 1;
  int lldb = 0, lkend = 0, lkc = 0, ldi = -1, li0 = 0;
  bool lrok = false;
  auto openL = [&]() {
    ldi = ddi;
    if (ddi >= 0) {
      const int row = di0 + warp * 8 + g;
      lrok = row < dM;
      lsk = dtA ? dlda : 1;                                   // A(row, k) = A[row*sr + k*sk]
      lAr = dA + (lrok ? (int64_t)row * (dtA ? 1 : dlda) : 0);
      lB = dB;
      lldb = dldb;
      // triangular records: op(A) lower (tri 1) ends the K range at the tile's last row, op(A)
      // upper (tri 3) starts it at the tile's first row; the skipped terms are structural zeros
      lkc = dtri == 3 ? (di0 / RG_K) * RG_K : 0;
      lkend = dtri == 1 ? min(dK, di0 + 64) : dK;
      li0 = di0;
    }
    fetchD();
  };
  // issue the loads of L's next chunk; returns its tag (descriptor id, row tile start, last chunk)
  auto issue = [&](double* a, int buf, int& tdi, int& ti0, bool& tlast) {
#pragma unroll
    for (int s = 0; s < RG_K / 4; ++s) {
      const int kg = lkc + 4 * s + t4;
      a[s] = (lrok && kg < lkend) ? __ldg(lAr + (int64_t)kg * lsk) : 0.0;
    }
    for (int e = tid; e < RG_K * NT8 * 8; e += NT) {
      const int kk = e / (NT8 * 8), c = e % (NT8 * 8);
      const bool ok = lkc + kk < lkend && c < N;
      cp_async8(&sB[buf][kk * LDB + c], lB + (ok ? (int64_t)(lkc + kk) * lldb + c : 0), ok);
    }
    cp_async_commit();
    tdi = ldi;
    ti0 = li0;
    lkc += RG_K;
    tlast = lkc >= lkend;
    if (tlast) openL();
  };
  fetchI();
  fetchD();
  openL();
  if (ldi < 0) return;
  double a0[RG_K / 4], a1[RG_K / 4];
  double acc[NT8][2];
#pragma unroll
  for (int y = 0; y < NT8; ++y) acc[y][0] = acc[y][1] = 0.0;
  int t0di, t0i0, t1di = -1, t1i0 = 0;
  bool t0last, t1last = false;
  issue(a0, 0, t0di, t0i0, t0last);
  int buf = 0;
  while (true) {
    const bool more = ldi >= 0;   // (uniform over the CTA: every thread walks the same list)
    if (more) {
      issue(a1, buf ^ 1, t1di, t1i0, t1last);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < RG_K / 4; ++s)
#pragma unroll
      for (int y = 0; y < NT8; ++y) dmma(acc[y][0], acc[y][1], a0[s], sB[buf][(4 * s + t4) * LDB + y * 8 + g]);
    if (t0last) {
      const GemmDesc* p = desc + t0di;
      const int row = t0i0 + warp * 8 + g;
      if (row < p->M) {
        const double alpha = p->alpha, beta = p->beta;
        double* crow = p->C + (int64_t)row * p->ldc;
#pragma unroll
        for (int y = 0; y < NT8; ++y)
#pragma unroll
          for (int z = 0; z < 2; ++z) {
            const int c = y * 8 + 2 * t4 + z;
            if (c < N) crow[c] = (beta == 0.0 ? 0.0 : beta * crow[c]) + alpha * acc[y][z];
          }
      }
#pragma unroll
      for (int y = 0; y < NT8; ++y) acc[y][0] = acc[y][1] = 0.0;
    }
    __syncthreads();
    if (!more) break;
#pragma unroll
    for (int s = 0; s < RG_K / 4; ++s) a0[s] = a1[s];
    t0di = t1di;
    t0i0 = t1i0;
    t0last = t1last;
    buf ^= 1;
  }
}

// Deep records (mean K >= 128): one item at a time per CTA, K in 64-deep chunks, two-stage
// operand prefetch inside the item; CTAs are scheduled by the hardware (grid-stride over the list).
constexpr int RGD_K = 64;
template <int NT8>
__global__ void __launch_bounds__(NT) k_rgemm_deep(const GemmDesc* desc, const int* w_desc, const int* w_tile, int nwork) {
  constexpr int LDB = NT8 * 8 + 4;
  __shared__ double sB[2][RGD_K * LDB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t4 = lane & 3;
  for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
    const GemmDesc d = desc[w_desc[w]];
    const int i0 = 64 * w_tile[w];
    const int row = i0 + warp * 8 + g;
    const bool rok = row < d.M;
    const int64_t sr = d.transA ? 1 : d.lda, sk = d.transA ? d.lda : 1;   // A(row, k) = A[row*sr + k*sk]
    const double* Ar = d.A + (rok ? (int64_t)row * sr : 0);
    double acc[NT8][2];
#pragma unroll
    for (int y = 0; y < NT8; ++y) acc[y][0] = acc[y][1] = 0.0;
    auto load_a = [&](double* a, int kc) {
#pragma unroll
      for (int s = 0; s < RGD_K / 4; ++s) {
        const int kg = kc + 4 * s + t4;
        a[s] = (rok && kg < d.K) ? ldg_pf(Ar + (int64_t)kg * sk) : 0.0;
      }
    };
    auto stage_b = [&](int buf, int kc) {
      for (int e = tid; e < RGD_K * NT8 * 8; e += NT) {
        const int kk = e / (NT8 * 8), c = e % (NT8 * 8);
        const bool ok = kc + kk < d.K && c < d.N;
        cp_async8(&sB[buf][kk * LDB + c], d.B + (ok ? (int64_t)(kc + kk) * d.ldb + c : 0), ok);
      }
      cp_async_commit();
    };
    double a0[RGD_K / 4], a1[RGD_K / 4];
    // triangular records: op(A) lower (tri 1) ends the K range at the tile's last row, op(A)
    // upper (tri 3) starts it at the tile's first row; the skipped terms are structural zeros
    const int kbeg = d.tri == 3 ? (i0 / RGD_K) * RGD_K : 0;
    const int kend = d.tri == 1 ? min(d.K, i0 + 64) : d.K;
    __syncthreads();   // previous work item's reads of sB are done
    load_a(a0, kbeg);
    stage_b(0, kbeg);
    int buf = 0;
    for (int kc = kbeg; kc < kend; kc += RGD_K) {
      const bool more = kc + RGD_K < kend;
      if (more) {
        load_a(a1, kc + RGD_K);
        stage_b(buf ^ 1, kc + RGD_K);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
#pragma unroll
      for (int s = 0; s < RGD_K / 4; ++s)
#pragma unroll
        for (int y = 0; y < NT8; ++y) dmma(acc[y][0], acc[y][1], a0[s], sB[buf][(4 * s + t4) * LDB + y * 8 + g]);
      __syncthreads();
#pragma unroll
      for (int s = 0; s < RGD_K / 4; ++s) a0[s] = a1[s];
      buf ^= 1;
    }
    if (rok) {
#pragma unroll
      for (int y = 0; y < NT8; ++y)
#pragma unroll
        for (int z = 0; z < 2; ++z) {
          const int c = y * 8 + 2 * t4 + z;
          if (c < d.N) {
            double* p = d.C + (int64_t)row * d.ldc + c;
            *p = (d.beta == 0.0 ? 0.0 : d.beta * *p) + d.alpha * acc[y][z];
          }
        }
    }
  }
}

// Deep records, 17..32 right-hand sides: both operands staged in shared memory by cp.async (a warp
// copies 256 contiguous bytes of one row of A per instruction, instead of fragment loads that
// touch eight rows each), K in 32-deep chunks through a 3-stage pipeline with one barrier per
// chunk; warps 4 (rows) x 2 (columns), each a 16 x 16 tile. The load/store unit work per DMMA is
// about half that of k_rgemm_deep, which was co-limiting with the DMMA pipe.
constexpr int RS_BK = 32, RS_STAGES = 3;
constexpr int RS_ALD_N = RS_BK + 4;   // A not transposed: sA[row][k]
constexpr int RS_ALD_T = 64 + 4;      // A transposed:     sA[k][row]
constexpr int RS_BLD = 32 + 4;        // sB[k][col]
constexpr int RS_ASZ = 64 * RS_ALD_N > RS_BK * RS_ALD_T ? 64 * RS_ALD_N : RS_BK * RS_ALD_T;
constexpr int RS_STAGE = RS_ASZ + RS_BK * RS_BLD;
constexpr size_t RS_SMEM = (size_t)RS_STAGES * RS_STAGE * sizeof(double);
__global__ void __launch_bounds__(NT, 2) k_rgemm_smem(const GemmDesc* __restrict__ desc, const int* __restrict__ w_desc,
                                                       const int* __restrict__ w_tile, int nwork) {
  extern __shared__ double smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 3, wn = warp >> 2, g = lane >> 2, t = lane & 3;
  for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
    const GemmDesc d = desc[w_desc[w]];
    const int i0 = 64 * w_tile[w];
    const int M = min(64, d.M - i0);
    if (M <= 0) continue;
    const int Kb = d.tri == 3 ? (i0 / RS_BK) * RS_BK : 0;
    const int Kt = d.tri == 1 ? min(d.K, i0 + 64) : d.K;
    const int nk = (Kt - Kb + RS_BK - 1) / RS_BK;
    auto load = [&](int st, int k0) {
      double* sA = smem + st * RS_STAGE;
      double* sB = sA + RS_ASZ;
#pragma unroll
      for (int q = 0; q < (64 * RS_BK) / NT; ++q) {
        const int e = tid + q * NT;
        if (d.transA) {   // op(A)(i,k) = A[k*lda + i]: a warp copies 32 consecutive rows of one k
          const int kk = e >> 6, r = e & 63;
          const bool ok = r < M && k0 + kk < Kt;
          cp_async8_pf(sA + kk * RS_ALD_T + r, d.A + (ok ? (int64_t)(k0 + kk) * d.lda + i0 + r : 0), ok);
        } else {          // A[i*lda + k]: a warp copies the 32 k of one row
          const int r = e >> 5, kk = e & 31;
          const bool ok = r < M && k0 + kk < Kt;
          cp_async8_pf(sA + r * RS_ALD_N + kk, d.A + (ok ? (int64_t)(i0 + r) * d.lda + k0 + kk : 0), ok);
        }
      }
#pragma unroll
      for (int q = 0; q < (RS_BK * 32) / NT; ++q) {
        const int e = tid + q * NT, kk = e >> 5, c = e & 31;
        const bool ok = k0 + kk < Kt && c < d.N;
        cp_async8(sB + kk * RS_BLD + c, d.B + (ok ? (int64_t)(k0 + kk) * d.ldb + c : 0), ok);
      }
    };
    double acc[2][2][2];
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
    __syncthreads();   // the previous item's readers of the stage buffers are done
#pragma unroll
    for (int st = 0; st < RS_STAGES - 1; ++st) {
      if (st < nk) load(st, Kb + st * RS_BK);
      cp_async_commit();
    }
    for (int kc = 0; kc < nk; ++kc) {
      cp_async_wait<RS_STAGES - 2>();   // chunk kc has landed (this thread's copies)
      __syncthreads();                  // ... everyone's; and chunk kc-1 is consumed: its stage is free
      if (kc + RS_STAGES - 1 < nk) load((kc + RS_STAGES - 1) % RS_STAGES, Kb + (kc + RS_STAGES - 1) * RS_BK);
      cp_async_commit();
      const double* sA = smem + (kc % RS_STAGES) * RS_STAGE;
      const double* sB = sA + RS_ASZ;
#pragma unroll
      for (int ks = 0; ks < RS_BK; ks += 4) {
        double af[2], bf[2];
#pragma unroll
        for (int x = 0; x < 2; ++x)
          af[x] = d.transA ? sA[(ks + t) * RS_ALD_T + wm * 16 + x * 8 + g] : sA[(wm * 16 + x * 8 + g) * RS_ALD_N + ks + t];
#pragma unroll
        for (int y = 0; y < 2; ++y) bf[y] = sB[(ks + t) * RS_BLD + wn * 16 + y * 8 + g];
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
          for (int y = 0; y < 2; ++y) dmma(acc[x][y][0], acc[x][y][1], af[x], bf[y]);
      }
    }
    cp_async_wait<0>();
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      const int r = wm * 16 + x * 8 + g;
      if (r < M) {
        double* crow = d.C + (int64_t)(i0 + r) * d.ldc;
#pragma unroll
        for (int y = 0; y < 2; ++y)
#pragma unroll
          for (int z = 0; z < 2; ++z) {
            const int c = wn * 16 + y * 8 + 2 * t + z;
            if (c < d.N) crow[c] = (d.beta == 0.0 ? 0.0 : d.beta * crow[c]) + d.alpha * acc[x][y][z];
          }
      }
    }
  }
}

// Batched GEMM, C[64-row tile, :] = beta*C + alpha*op(A)[rows, :] B: the N columns in 64-wide
// chunks (one 64 x 64 output tile at a time), K streamed in 16-wide chunks through a 3-stage
// cp.async pipeline, each warp a 16 x 32 DMMA tile (2 x 4 m8n8k4 fragments).
constexpr int BG_BK = 16, BG_ALD = BG_BK + 4, BG_BLD = 64 + 4, BG_STAGES = 3;
constexpr int BG_STAGE = 64 * BG_ALD + BG_BK * BG_BLD;
constexpr size_t BG_SMEM = (size_t)BG_STAGES * BG_STAGE * sizeof(double);
__global__ void __launch_bounds__(NT, 2) k_bgemm(const GemmDesc* desc, const int* w_desc, const int* w_tile,
                                                  int nwork) {
  extern __shared__ double smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 3, wn = warp >> 2, g = lane >> 2, t = lane & 3;
  for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
    const GemmDesc d = desc[w_desc[w]];
    const int i0 = 64 * w_tile[w];
    const int M = min(64, d.M - i0);
    if (M <= 0) continue;
    for (int j0 = 0; j0 < d.N; j0 += 64) {
      const int N = min(64, d.N - j0);
      // triangular operands: the K range ends at the tile's last row (op(A) lower) or column
      // (B upper); the terms beyond are structural zeros
      const int Kt = d.tri == 1 ? min(d.K, i0 + 64) : (d.tri == 2 ? min(d.K, j0 + 64) : d.K);
      auto load = [&](int st, int k0) {
        double* sA = smem + st * BG_STAGE;
        double* sB = sA + 64 * BG_ALD;
#pragma unroll
        for (int q = 0; q < (64 * BG_BK) / NT; ++q) {
          const int e = tid + q * NT;
          int r, kk;
          if (d.transA) {   // op(A)(i,k) = A[k*lda + i]: coalesce along i
            kk = e / 64;
            r = e % 64;
          } else {          // A[i*lda + k]
            r = e / BG_BK;
            kk = e % BG_BK;
          }
          const int gi = i0 + r, gk = k0 + kk;
          const bool ok = r < M && gk < Kt;
          const double* src = d.transA ? d.A + (ok ? (int64_t)gk * d.lda + gi : 0)
                                       : d.A + (ok ? (int64_t)gi * d.lda + gk : 0);
          cp_async8(sA + r * BG_ALD + kk, src, ok);
        }
#pragma unroll
        for (int q = 0; q < (BG_BK * 64) / NT; ++q) {
          const int e = tid + q * NT, kk = e / 64, c = e % 64;
          const int gk = k0 + kk;
          const bool ok = gk < Kt && c < N;
          cp_async8(sB + kk * BG_BLD + c, d.B + (ok ? (int64_t)gk * d.ldb + j0 + c : 0), ok);
        }
        cp_async_commit();
      };
      double acc[2][4][2];
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
      const int Kb = d.tri == 3 ? (i0 / BG_BK) * BG_BK : 0;
      const int nk = (Kt - Kb + BG_BK - 1) / BG_BK;
      __syncthreads();   // previous tile's readers of the stage buffers are done
      if (nk > 0) load(0, Kb);
      if (nk > 1) load(1, Kb + BG_BK);
      for (int kc = 0; kc < nk; ++kc) {
        if (kc + 2 < nk) {
          load((kc + 2) % BG_STAGES, Kb + (kc + 2) * BG_BK);
          cp_async_wait<2>();
        } else if (kc + 1 < nk) {
          cp_async_wait<1>();
        } else {
          cp_async_wait<0>();
        }
        __syncthreads();
        const double* sA = smem + (kc % BG_STAGES) * BG_STAGE;
        const double* sB = sA + 64 * BG_ALD;
#pragma unroll
        for (int ks = 0; ks < BG_BK; ks += 4) {
          double af[2], bf[4];
#pragma unroll
          for (int x = 0; x < 2; ++x) af[x] = sA[(wm * 16 + x * 8 + g) * BG_ALD + ks + t];
#pragma unroll
          for (int y = 0; y < 4; ++y) bf[y] = sB[(ks + t) * BG_BLD + wn * 32 + y * 8 + g];
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
            const int r = wm * 16 + x * 8 + g, c = wn * 32 + y * 8 + 2 * t + z;
            if (r < M && c < N) {
              double* p = d.C + (int64_t)(i0 + r) * d.ldc + j0 + c;
              *p = (d.beta == 0.0 ? 0.0 : d.beta * *p) + d.alpha * acc[x][y][z];
            }
          }
    }
  }
}

// gather / scatter of DOF rows for a list of index segments: Y[seg_dst + e] <-> x[idx[seg_src + e]]
// (one warp per segment, grid-stride over segments)
__global__ void k_rows(double* Y, double* x, const int* idx, const int64_t* seg_src, const int64_t* seg_dst,
                       const int* seg_len, int nseg, int k, int to_x, int chunks) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int sgi = blockIdx.x * wpb + (threadIdx.x >> 5); sgi < nseg; sgi += gridDim.x * wpb) {
    const int* id = idx + seg_src[sgi];
    double* y = Y + seg_dst[sgi] * k;
    if (k == 32) {   // lane = right-hand side, 8 rows in flight (no index division)
      const int nr = seg_len[sgi];
      for (int r0 = 0; r0 < nr; r0 += 8) {
        int rid[8];
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) rid[u] = r0 + u < nr ? __ldg(id + r0 + u) : 0;
        if (to_x) {
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = r0 + u < nr ? y[(int64_t)(r0 + u) * 32 + lane] : 0.0;
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (r0 + u < nr) x[(int64_t)rid[u] * 32 + lane] = v[u];
        } else {
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = r0 + u < nr ? x[(int64_t)rid[u] * 32 + lane] : 0.0;
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (r0 + u < nr) y[(int64_t)(r0 + u) * 32 + lane] = v[u];
        }
      }
      continue;
    }
    const int64_t n = (int64_t)seg_len[sgi] * k;
    for (int64_t e = lane; e < n; e += 32) {
      double* px = x + (int64_t)id[e / k] * k + e % k;
      if (to_x) *px = y[e];
      else y[e] = *px;
    }
  }
  (void)chunks;
}

// ---------------------------------------------------------------------------
// Level transition: carry the surviving live matrix into the next grouping.
// ---------------------------------------------------------------------------
// One CTA per row chunk of a new block. Every (source group of G) x (source group of H) pair
// resolves to an old block (or none) once, in a shared-memory table; rows then run per warp
// and columns per lane.
struct RepackEnt {
  long long base;   // old block offset, -1: no block (zero)
  int rs, cs;       // element (pi, pj) at base + pi*rs + pj*cs
};
__global__ void __launch_bounds__(NT) k_repack(RepackArgs ra) {
  extern __shared__ double smem[];
  RepackEnt* tab = reinterpret_cast<RepackEnt*>(smem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = NT / 32;
  const int b = ra.w_blk[blockIdx.x], row0 = ra.w_row0[blockIdx.x], nrow = ra.w_nrow[blockIdx.x];
  const int G = ra.nbg[b], H = ra.nbh[b];
  const int64_t oG = ra.ngoff[G], oH = ra.ngoff[H];
  const int cols = (int)(ra.ngoff[H + 1] - oH);
  const int64_t sG = ra.nsrcl_off[G], sH = ra.nsrcl_off[H];
  const int nH = (int)(ra.nsrcl_off[H + 1] - sH);
  const int nt = (int)(ra.nsrcl_off[G + 1] - sG) * nH;
  double* dst = ra.npool + ra.nboff[b];
  if ((int64_t)nt * 8 > (int64_t)nrow * cols) {
    // small chunk: resolve the old block per element
    for (int i = row0 + warp; i < row0 + nrow; i += nw) {
      const int og = ra.nsrcl[sG + ra.nsrc_local[oG + i]];
      const int64_t pi = ra.nsrc_pos[oG + i];
      double* drow = dst + (int64_t)i * cols;
      for (int j = lane; j < cols; j += 32) {
        const int oh = ra.nsrcl[sH + ra.nsrc_local[oH + j]];
        const int64_t pj = ra.nsrc_pos[oH + j];
        double v = 0.0;
        if (og <= oh) {
          const int blk = find_blk(ra.oadj_off, ra.oadj_nbr, ra.oadj_blk, og, oh);
          if (blk >= 0) v = __ldg(ra.opool + ra.oboff[blk] + pi * ra.ogsize[oh] + pj);
        } else {
          const int blk = find_blk(ra.oadj_off, ra.oadj_nbr, ra.oadj_blk, oh, og);
          if (blk >= 0) v = __ldg(ra.opool + ra.oboff[blk] + pj * ra.ogsize[og] + pi);
        }
        drow[j] = v;
      }
    }
    return;
  }
  for (int e = tid; e < nt; e += NT) {
    const int og = ra.nsrcl[sG + e / nH], oh = ra.nsrcl[sH + e % nH];
    RepackEnt t{-1, 0, 0};
    if (og <= oh) {
      const int blk = find_blk(ra.oadj_off, ra.oadj_nbr, ra.oadj_blk, og, oh);
      if (blk >= 0) t = RepackEnt{(long long)ra.oboff[blk], ra.ogsize[oh], 1};
    } else {
      const int blk = find_blk(ra.oadj_off, ra.oadj_nbr, ra.oadj_blk, oh, og);
      if (blk >= 0) t = RepackEnt{(long long)ra.oboff[blk], 1, ra.ogsize[og]};
    }
    tab[e] = t;
  }
  __syncthreads();
  for (int i = row0 + warp; i < row0 + nrow; i += nw) {
    const RepackEnt* trow = tab + ra.nsrc_local[oG + i] * nH;
    const int64_t pi = ra.nsrc_pos[oG + i];
    double* drow = dst + (int64_t)i * cols;
    for (int j = lane; j < cols; j += 32) {
      const RepackEnt t = trow[ra.nsrc_local[oH + j]];
      const int64_t pj = ra.nsrc_pos[oH + j];
      drow[j] = t.base >= 0 ? __ldg(ra.opool + t.base + pi * t.rs + pj * t.cs) : 0.0;
    }
  }
}

// ---------------------------------------------------------------------------
// Forward replay: F x = G G^T x (oracle/phif.py _gt/_g). Same records as the
// inverse replay, multiplied instead of solved. One CTA per record; records of one launch own
// disjoint DOF sets. Record panels are row-major with a zero strict upper triangle in L, so
// G^T of a cell is one transposed product P^T [x_I; x_B] and G is P x_I.
// ---------------------------------------------------------------------------
// y[col] = sum_rho P[rho][col] * v(rho) over rows [0, nr) of a row-major panel (ld = ncol):
// threads along columns (coalesced), v(rho) broadcast
template <typename VF>
__device__ __forceinline__ double colsum(const double* P, int ld, int nr, int col, VF v) {
  double a = 0.0;
  for (int rho = 0; rho < nr; ++rho) a += P[(int64_t)rho * ld + col] * v(rho);
  return a;
}
__device__ __forceinline__ double rowdot(const double* Prow, int n, const double* x, const int* idx, int k, int c) {
  const int lane = threadIdx.x & 31;
  double a = 0.0;
  for (int i = lane; i < n; i += 32) a += Prow[i] * x[(int64_t)idx[i] * k + c];
  return warp_sum(a);
}

// cells: up = G^T (x_I <- L^T x_I + X x_B), else G (x_B += X^T x_I via wbuf, x_I <- L x_I)
__global__ void __launch_bounds__(NT) k_fwd_cell(ApplyCellArgs a, double* x, int k, int up) {
  const int t = blockIdx.x;
  const int n = a.n[t], b = a.b[t];
  const int* I = a.I + a.I_off[t];
  const int* B = a.B + a.B_off[t];
  const double* P = a.rec + a.P_off[t];
  double* Y = a.work + a.work_off[t] * k;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = NT / 32;
  for (int c = 0; c < k; ++c) {
    if (up) {
      for (int i = tid; i < n; i += NT)
        Y[i] = colsum(P, n, n + b, i, [&](int rho) {
          return x[(int64_t)(rho < n ? I[rho] : B[rho - n]) * k + c];
        });
      __syncthreads();
      for (int i = tid; i < n; i += NT) x[(int64_t)I[i] * k + c] = Y[i];
    } else {
      for (int rho = warp; rho < n + b; rho += nw) {
        const double z = rowdot(P + (int64_t)rho * n, n, x, I, k, c);
        if (lane == 0) {
          if (rho < n) Y[rho] = z;
          else a.wbuf[(a.B_off[t] + rho - n) * k + c] = -z;   // the reduction subtracts
        }
      }
      __syncthreads();
      for (int i = tid; i < n; i += NT) x[(int64_t)I[i] * k + c] = Y[i];
    }
    __syncthreads();
  }
}

// block-Jacobi groups: up = G^T (x_I <- L^T x_I), else G (x_I <- L x_I); record [L ; L^-T]
__global__ void __launch_bounds__(NT) k_fwd_prec(ApplyPrecArgs a, double* x, int k, int up) {
  const int t = blockIdx.x;
  const int n = a.n[t];
  const int* I = a.I + a.I_off[t];
  const double* L = a.rec + a.L_off[t];
  double* Y = a.work + a.work_off[t] * k;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = NT / 32;
  for (int c = 0; c < k; ++c) {
    if (up) {
      for (int i = tid; i < n; i += NT)
        Y[i] = colsum(L, n, n, i, [&](int rho) { return x[(int64_t)I[rho] * k + c]; });
    } else {
      for (int rho = warp; rho < n; rho += nw) {
        const double z = rowdot(L + (int64_t)rho * n, n, x, I, k, c);
        if (lane == 0) Y[rho] = z;
      }
    }
    __syncthreads();
    for (int i = tid; i < n; i += NT) x[(int64_t)I[i] * k + c] = Y[i];
    __syncthreads();
  }
}

// separators (records T (r x kt) and [L~ ; X~^T ; L~^-T]):
//  up (G^T): x_S += T x_R ; x_R <- L~^T x_R + X~ x_S
//  down (G): x_S += X~^T x_R ; x_R <- L~ x_R ; x_R += T^T x_S
__global__ void __launch_bounds__(NT) k_fwd_skel(ApplySkelArgs a, double* x, int k, int up) {
  const int t = blockIdx.x;
  const int r = a.r[t], kt = a.kt[t];
  if (kt == 0) return;
  const int* S = a.S + a.S_off[t];
  const int* R = a.R + a.R_off[t];
  const double* T = a.rec + a.T_off[t];
  const double* P = a.rec + a.P_off[t];
  double* Y = a.work + a.work_off[t] * k;   // r + kt per right-hand side
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = NT / 32;
  for (int c = 0; c < k; ++c) {
    if (up) {
      for (int q = warp; q < r; q += nw) {
        const double z = rowdot(T + (int64_t)q * kt, kt, x, R, k, c);
        if (lane == 0) Y[q] = x[(int64_t)S[q] * k + c] + z;
      }
      __syncthreads();
      for (int q = tid; q < r; q += NT) x[(int64_t)S[q] * k + c] = Y[q];
      __syncthreads();
      for (int i = tid; i < kt; i += NT)
        Y[r + i] = colsum(P, kt, kt + r, i, [&](int rho) {
          return rho < kt ? x[(int64_t)R[rho] * k + c] : Y[rho - kt];
        });
      __syncthreads();
      for (int i = tid; i < kt; i += NT) x[(int64_t)R[i] * k + c] = Y[r + i];
    } else {
      for (int rho = warp; rho < kt + r; rho += nw) {
        const double z = rowdot(P + (int64_t)rho * kt, kt, x, R, k, c);
        if (lane == 0) {
          if (rho < kt) Y[r + rho] = z;
          else Y[rho - kt] = x[(int64_t)S[rho - kt] * k + c] + z;
        }
      }
      __syncthreads();
      for (int q = tid; q < r; q += NT) x[(int64_t)S[q] * k + c] = Y[q];
      for (int i = tid; i < kt; i += NT) {
        double z = Y[r + i];
        for (int q = 0; q < r; ++q) z += T[(int64_t)q * kt + i] * Y[q];
        x[(int64_t)R[i] * k + c] = z;
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Record replay (apply F^-1, G^-1, G^-T)
// x is N x k row-major (DOF-major, right-hand sides contiguous).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void gather_rows(double* Y, const double* x, const int* idx, int n, int k) {
  for (int64_t e = threadIdx.x; e < (int64_t)n * k; e += NT) Y[e] = x[(int64_t)idx[e / k] * k + e % k];
}
__device__ __forceinline__ void scatter_rows(double* x, const double* Y, const int* idx, int n, int k) {
  for (int64_t e = threadIdx.x; e < (int64_t)n * k; e += NT) x[(int64_t)idx[e / k] * k + e % k] = Y[e];
}

__global__ void __launch_bounds__(NT) k_apply_cell(ApplyCellArgs a, double* x, int k, int up) {
  extern __shared__ double smem[];
  const int t = a.list ? a.list[blockIdx.x] : blockIdx.x;
  const int n = a.n[t], b = a.b[t];
  const int* I = a.I + a.I_off[t];
  const int* B = a.B + a.B_off[t];
  const double* P = a.rec + a.P_off[t];
  double* Y = a.work + a.work_off[t] * k;
  gather_rows(Y, x, I, n, k);
  __syncthreads();
  if (up) {
    cta_trsm_left(P, n, n, Y, k, k, false, smem);
    scatter_rows(x, Y, I, n, k);
    if (b > 0)
      cta_gemm<false, false>(b, k, n, 1.0, P + (int64_t)n * n, n, Y, k, 0.0, a.wbuf + a.B_off[t] * k, k, false,
                             smem + GEMM_OFF);
  } else {
    if (b > 0) {
      double* Z = Y + (int64_t)n * k;
      gather_rows(Z, x, B, b, k);
      __syncthreads();
      cta_gemm<true, false>(n, k, b, -1.0, P + (int64_t)n * n, n, Z, k, 1.0, Y, k, false, smem + GEMM_OFF);
    }
    cta_trsm_left(P, n, n, Y, k, k, true, smem);
    scatter_rows(x, Y, I, n, k);
  }
}

// x_B -= sum of cell contributions, fixed cell order per boundary DOF
__global__ void k_apply_reduce(const int* dof, const int64_t* off, const int* rows, const double* wbuf, int nd,
                               double* x, int k) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)nd * k) return;
  const int i = (int)(e / k), c = (int)(e % k);
  double s = x[(int64_t)dof[i] * k + c];
  for (int64_t q = off[i]; q < off[i + 1]; ++q) s -= wbuf[(int64_t)rows[q] * k + c];
  x[(int64_t)dof[i] * k + c] = s;
}

// small block-Jacobi records: one warp per group, dense product with the stored L^-T
__global__ void k_apply_prec_tiny(ApplyPrecArgs a, double* x, int k, int up, int ldn) {
  // one warp per group (|g| < APPLY_BIG): the group's rows are staged in shared memory, then
  // y = L^-1 x (up) or L^-T x (down) from the stored L^-T, written straight back to x
  extern __shared__ double smem[];
  const int wpc = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wg = blockIdx.x * wpc + warp;
  if (wg >= a.r) return;
  const int t = a.list ? a.list[wg] : wg;
  const int n = a.n[t];
  const int* I = a.I + a.I_off[t];
  const double* LiT = a.rec + a.L_off[t] + (int64_t)n * n;
  if (k == 32) {   // 32 right-hand sides: lane = right-hand side, no index division
    double* Y = ldn > 0 ? smem + (size_t)warp * ldn * 32 : a.work + a.work_off[t] * 32;
    for (int i = 0; i < n; ++i) Y[i * 32 + lane] = x[(int64_t)I[i] * 32 + lane];
    for (int i = 0; i < n; ++i) {
      double s = 0.0;
      if (up)
        for (int j = 0; j <= i; ++j) s = __fma_rn(__ldg(LiT + (int64_t)j * n + i), Y[j * 32 + lane], s);
      else
        for (int j = i; j < n; ++j) s = __fma_rn(__ldg(LiT + (int64_t)i * n + j), Y[j * 32 + lane], s);
      x[(int64_t)I[i] * 32 + lane] = s;
    }
    return;
  }
  if (ldn > 0) {   // few right-hand sides: stage the rows, write straight back
    double* Y = smem + (size_t)warp * ldn * k;
    for (int e = lane; e < n * k; e += 32) Y[e] = x[(int64_t)I[e / k] * k + e % k];
    __syncwarp();
    for (int e = lane; e < n * k; e += 32) {
      const int i = e / k, c = e % k;
      double s = 0.0;
      if (up)   // y = L^-1 x = (L^-T)^T x, L^-T upper triangular
        for (int j = 0; j <= i; ++j) s += __ldg(LiT + (int64_t)j * n + i) * Y[j * k + c];
      else      // y = L^-T x
        for (int j = i; j < n; ++j) s += __ldg(LiT + (int64_t)i * n + j) * Y[j * k + c];
      x[(int64_t)I[i] * k + c] = s;
    }
    return;
  }
  // many right-hand sides: lanes along the right-hand sides read x directly (coalesced),
  // results buffered in the record's workspace
  double* Yw = a.work + a.work_off[t] * k;
  for (int e = lane; e < n * k; e += 32) {
    const int i = e / k, c = e % k;
    double s = 0.0;
    if (up)
      for (int j = 0; j <= i; ++j) s += __ldg(LiT + (int64_t)j * n + i) * x[(int64_t)I[j] * k + c];
    else
      for (int j = i; j < n; ++j) s += __ldg(LiT + (int64_t)i * n + j) * x[(int64_t)I[j] * k + c];
    Yw[e] = s;
  }
  __syncwarp();
  for (int e = lane; e < n * k; e += 32) x[(int64_t)I[e / k] * k + e % k] = Yw[e];
}

__global__ void __launch_bounds__(NT) k_apply_prec(ApplyPrecArgs a, double* x, int k, int up) {
  extern __shared__ double smem[];
  const int t = a.list ? a.list[blockIdx.x] : blockIdx.x;
  const int n = a.n[t];
  const int* I = a.I + a.I_off[t];
  double* Y = a.work + a.work_off[t] * k;
  gather_rows(Y, x, I, n, k);
  __syncthreads();
  cta_trsm_left(a.rec + a.L_off[t], n, n, Y, k, k, !up, smem);
  scatter_rows(x, Y, I, n, k);
}

// Small separators (|g| <= 64): one warp per record. The warp stages its rows (skeleton,
// redundant, and a k~-row temporary) in shared memory, then with the stored L~^-T:
//   up:   Y_r -= T^T Y_s ; Z = L~^-1 Y_r ; Y_s -= X~^T Z
//   down: Y_r -= X~ Y_s  ; Z = L~^-T Y_r ; Y_s -= T Z
// (oracle/phif.py _up/_down, same as k_apply_skel); lanes run over (row, rhs) pairs.
__global__ void __launch_bounds__(128) k_apply_skel_warp(ApplySkelArgs a, const int* list, int n, double* x, int k,
                                                         int up, int ldrows) {
  extern __shared__ double smem[];
  const int wpc = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int idx = blockIdx.x * wpc + warp;
  if (idx >= n) return;
  const int t = list[idx];
  const int r = a.r[t], kt = a.kt[t];
  const int* S = a.S + a.S_off[t];
  const int* R = a.R + a.R_off[t];
  const double* T = a.rec + a.T_off[t];                     // r x kt
  const double* PB = a.rec + a.P_off[t] + (int64_t)kt * kt;  // X~^T: r x kt
  const double* LiT = PB + (int64_t)r * kt;                 // L~^-T: kt x kt (upper)
  double* Ys = smem + (size_t)warp * ldrows * k;
  double* Yr = Ys + (size_t)r * k;
  double* Z = Yr + (size_t)kt * k;
  if (k == 32) {   // lane = right-hand side: every lane works on its own column (no warp sync)
    // gathers: indices one per lane (shuffled), 8 row loads in flight before their stores
    for (int q0 = 0; q0 < r; q0 += 32) {
      const int myS = q0 + lane < r ? S[q0 + lane] : 0;
      for (int q1 = 0; q1 < min(32, r - q0); q1 += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int gi = __shfl_sync(0xffffffffu, myS, (q1 + u) & 31);
          v[u] = q0 + q1 + u < r ? x[(int64_t)gi * 32 + lane] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (q0 + q1 + u < r) Ys[(q0 + q1 + u) * 32 + lane] = v[u];
      }
    }
    for (int j0 = 0; j0 < kt; j0 += 32) {
      const int myR = j0 + lane < kt ? R[j0 + lane] : 0;
      for (int j1 = 0; j1 < min(32, kt - j0); j1 += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int gi = __shfl_sync(0xffffffffu, myR, (j1 + u) & 31);
          v[u] = j0 + j1 + u < kt ? x[(int64_t)gi * 32 + lane] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (j0 + j1 + u < kt) Yr[(j0 + j1 + u) * 32 + lane] = v[u];
      }
    }
    const double* M1 = up ? T : PB;    // b_R -= M1^T b_S
    const double* M3 = up ? PB : T;    // b_S -= M3 z
    for (int j0 = 0; j0 < kt; j0 += 4) {   // four outputs per pass: independent FMA chains
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 4
      for (int q = 0; q < r; ++q) {
        const double y = Ys[q * 32 + lane];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (j0 + u < kt) acc[u] = __fma_rn(__ldg(M1 + (int64_t)q * kt + j0 + u), y, acc[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (j0 + u < kt) Yr[(j0 + u) * 32 + lane] -= acc[u];
    }
    for (int i = 0; i < kt; ++i) {
      double sacc = 0.0;
      if (up) {
#pragma unroll 8
        for (int j = 0; j <= i; ++j) sacc = __fma_rn(__ldg(LiT + (int64_t)j * kt + i), Yr[j * 32 + lane], sacc);
      } else {
#pragma unroll 8
        for (int j = i; j < kt; ++j) sacc = __fma_rn(__ldg(LiT + (int64_t)i * kt + j), Yr[j * 32 + lane], sacc);
      }
      Z[i * 32 + lane] = sacc;
    }
    for (int q0 = 0; q0 < r; q0 += 4) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 4
      for (int i = 0; i < kt; ++i) {
        const double z = Z[i * 32 + lane];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (q0 + u < r) acc[u] = __fma_rn(__ldg(M3 + (int64_t)(q0 + u) * kt + i), z, acc[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (q0 + u < r) x[(int64_t)S[q0 + u] * 32 + lane] = Ys[(q0 + u) * 32 + lane] - acc[u];
    }
    for (int i = 0; i < kt; ++i) x[(int64_t)R[i] * 32 + lane] = Z[i * 32 + lane];
    return;
  }
  for (int e = lane; e < r * k; e += 32) Ys[e] = x[(int64_t)S[e / k] * k + e % k];
  for (int e = lane; e < kt * k; e += 32) Yr[e] = x[(int64_t)R[e / k] * k + e % k];
  __syncwarp();
  if (up) {
    for (int e = lane; e < kt * k; e += 32) {
      const int j = e / k, c = e % k;
      double s = 0.0;
      for (int q = 0; q < r; ++q) s += __ldg(T + (int64_t)q * kt + j) * Ys[q * k + c];
      Yr[e] -= s;
    }
    __syncwarp();
    for (int e = lane; e < kt * k; e += 32) {
      const int i = e / k, c = e % k;
      double s = 0.0;
      for (int j = 0; j <= i; ++j) s += __ldg(LiT + (int64_t)j * kt + i) * Yr[j * k + c];
      Z[e] = s;
    }
    __syncwarp();
    for (int e = lane; e < r * k; e += 32) {
      const int q = e / k, c = e % k;
      double s = 0.0;
      for (int i = 0; i < kt; ++i) s += __ldg(PB + (int64_t)q * kt + i) * Z[i * k + c];
      Ys[e] -= s;
    }
  } else {
    for (int e = lane; e < kt * k; e += 32) {
      const int j = e / k, c = e % k;
      double s = 0.0;
      for (int q = 0; q < r; ++q) s += __ldg(PB + (int64_t)q * kt + j) * Ys[q * k + c];
      Yr[e] -= s;
    }
    __syncwarp();
    for (int e = lane; e < kt * k; e += 32) {
      const int i = e / k, c = e % k;
      double s = 0.0;
      for (int j = i; j < kt; ++j) s += __ldg(LiT + (int64_t)i * kt + j) * Yr[j * k + c];
      Z[e] = s;
    }
    __syncwarp();
    for (int e = lane; e < r * k; e += 32) {
      const int q = e / k, c = e % k;
      double s = 0.0;
      for (int j = 0; j < kt; ++j) s += __ldg(T + (int64_t)q * kt + j) * Z[j * k + c];
      Ys[e] -= s;
    }
  }
  __syncwarp();
  for (int e = lane; e < r * k; e += 32) x[(int64_t)S[e / k] * k + e % k] = Ys[e];
  for (int e = lane; e < kt * k; e += 32) x[(int64_t)R[e / k] * k + e % k] = Z[e];
}

// ---------------------------------------------------------------------------
// Warp-level DMMA replay of the small records for 32 right-hand sides (one warp per record).
// The record matrices are read straight from global memory as m8n8k4 A fragments (coalesced,
// every element once, all loads of a row tile in flight together); the right-hand-side rows are
// staged in shared memory (row stride TW_LD: conflict-free B fragments). No FMA dependency chain
// and no broadcast loads, which bound the lane-per-RHS kernels above.
// ---------------------------------------------------------------------------
constexpr int TW_LD = 36;
// acc(i, 0:32) = sum_j M(i, j) sB[j][0:32] for i < m, j in the row tile's K range:
//   M(i, j) = TRANS ? Mg[j*ld + i] : Mg[i*ld + j];  tri 0: j < kk; 1 (lower): j < min(kk, 8mt+8);
//   3 (upper): j >= 8mt. sB rows up to the next multiple of 4 of kk must be finite (zero padded).
// epi(row, ok, acc) receives each finished 8-row tile: lane (g, t4) holds row 8mt+g, columns
// 8y + 2 t4 + {0, 1} in acc[y][0..1].
template <bool TRANS, typename Epi>
__device__ __forceinline__ void warp_mm32(const double* __restrict__ Mg, int ld, int m, int kk, int tri,
                                          const double* sB, Epi epi) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  const int nmt = (m + 7) >> 3;
  if (nmt == 0) return;
  auto klo = [&](int mt) { return tri == 3 ? 8 * mt : 0; };
  auto khi = [&](int mt) { return tri == 1 ? min(kk, 8 * mt + 8) : kk; };
  auto load = [&](double* a, int mt, int k0) {
    const int row = 8 * mt + g, hi = khi(mt);
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int kg = k0 + 4 * s + t4;
      a[s] = (row < m && kg < hi) ? __ldg(TRANS ? Mg + (int64_t)kg * ld + row : Mg + (int64_t)row * ld + kg) : 0.0;
    }
  };
  double a0[8], a1[8], acc[4][2];
#pragma unroll
  for (int y = 0; y < 4; ++y) acc[y][0] = acc[y][1] = 0.0;
  int mt = 0, k0 = klo(0);
  load(a0, mt, k0);
  while (mt < nmt) {
    int nm = mt, nk = k0 + 32;
    if (nk >= khi(mt)) {
      nm = mt + 1;
      nk = klo(nm);
    }
    if (nm < nmt) load(a1, nm, nk);
    const int hi = khi(mt);
#pragma unroll
    for (int s = 0; s < 8; ++s)
      if (k0 + 4 * s < hi) {   // (warp-uniform)
        const double* b = sB + (k0 + 4 * s + t4) * TW_LD + g;
#pragma unroll
        for (int y = 0; y < 4; ++y) dmma(acc[y][0], acc[y][1], a0[s], b[8 * y]);
      }
    if (nm != mt) {
      epi(8 * mt + g, 8 * mt + g < m, acc);
#pragma unroll
      for (int y = 0; y < 4; ++y) acc[y][0] = acc[y][1] = 0.0;
    }
#pragma unroll
    for (int s = 0; s < 8; ++s) a0[s] = a1[s];
    mt = nm;
    k0 = nk;
  }
}

// stage rows x[idx[i]] (i < n) of a 32-column block into sY (row stride TW_LD), zero rows up to
// the next multiple of 4; lane = column, 8 row loads in flight
__device__ __forceinline__ void warp_stage32(double* sY, const double* x, const int* __restrict__ idx, int n) {
  const int lane = threadIdx.x & 31;
  for (int q0 = 0; q0 < n; q0 += 32) {
    const int mine = q0 + lane < n ? __ldg(idx + q0 + lane) : 0;
    const int lim = min(32, n - q0);
    for (int q1 = 0; q1 < lim; q1 += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int gi = __shfl_sync(0xffffffffu, mine, (q1 + u) & 31);
        v[u] = q1 + u < lim ? x[(int64_t)gi * 32 + lane] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (q1 + u < lim) sY[(q0 + q1 + u) * TW_LD + lane] = v[u];
    }
  }
  for (int i = n; i < ((n + 3) & ~3); ++i) sY[i * TW_LD + lane] = 0.0;
}

// small cells (n <= 32, b <= 64: the level-0 cells of a 3D grid), 32 right-hand sides; record panel
// [L ; X^T ; L^-T] (row stride n):
//   up:   Z = L^-1 x_I ; x_I <- Z ; wbuf rows of the cell <- X^T Z   (k_apply_reduce subtracts them)
//   down: Y = x_I - X x_B ; x_I <- L^-T Y
// Replaces gather -> two replay GEMMs -> scatter through the global workspace by one pass.
__global__ void __launch_bounds__(128) k_apply_cell_mma(ApplyCellArgs a, double* x, int up, int nrows, int ldrows) {
  extern __shared__ double smem[];
  const int wpc = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31, t4 = lane & 3;
  const int t = blockIdx.x * wpc + warp;
  if (t >= a.p) return;
  const int n = a.n[t], b = a.b[t];
  const int* I = a.I + a.I_off[t];
  const int* B = a.B + a.B_off[t];
  const double* P = a.rec + a.P_off[t];
  const double* XT = P + (int64_t)n * n;         // b x n
  const double* LiT = XT + (int64_t)b * n;       // n x n (upper)
  double* sY = smem + (size_t)warp * ldrows * TW_LD;
  double* s2 = sY + (size_t)nrows * TW_LD;       // Z (up) or x_B (down)
  warp_stage32(sY, x, I, n);
  if (up) {
    for (int i = n; i < ((n + 3) & ~3); ++i) s2[i * TW_LD + lane] = 0.0;
    __syncwarp();
    warp_mm32<true>(LiT, n, n, n, 1, sY, [&](int row, bool ok, double (&acc)[4][2]) {
      if (!ok) return;
      double* z = s2 + row * TW_LD + 2 * t4;
      double* xr = x + (int64_t)__ldg(I + row) * 32 + 2 * t4;
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        z[8 * y] = acc[y][0];
        z[8 * y + 1] = acc[y][1];
        *reinterpret_cast<double2*>(xr + 8 * y) = make_double2(acc[y][0], acc[y][1]);
      }
    });
    __syncwarp();
    double* wb = a.wbuf + a.B_off[t] * 32;
    warp_mm32<false>(XT, n, b, n, 0, s2, [&](int row, bool ok, double (&acc)[4][2]) {
      if (!ok) return;
      double* wr = wb + (int64_t)row * 32 + 2 * t4;
#pragma unroll
      for (int y = 0; y < 4; ++y) *reinterpret_cast<double2*>(wr + 8 * y) = make_double2(acc[y][0], acc[y][1]);
    });
  } else {
    warp_stage32(s2, x, B, b);
    __syncwarp();
    warp_mm32<true>(XT, n, n, b, 0, s2, [&](int row, bool ok, double (&acc)[4][2]) {
      if (!ok) return;
      double* yr = sY + row * TW_LD + 2 * t4;
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        yr[8 * y] -= acc[y][0];
        yr[8 * y + 1] -= acc[y][1];
      }
    });
    __syncwarp();
    warp_mm32<false>(LiT, n, n, n, 3, sY, [&](int row, bool ok, double (&acc)[4][2]) {
      if (!ok) return;
      double* xr = x + (int64_t)__ldg(I + row) * 32 + 2 * t4;
#pragma unroll
      for (int y = 0; y < 4; ++y) *reinterpret_cast<double2*>(xr + 8 * y) = make_double2(acc[y][0], acc[y][1]);
    });
  }
}

// block-Jacobi records (|g| < APPLY_BIG), 32 right-hand sides: x_g <- L^-1 x_g (up) / L^-T x_g
__global__ void __launch_bounds__(256) k_apply_prec_mma(ApplyPrecArgs a, double* x, int up, int ldn) {
  extern __shared__ double smem[];
  const int wpc = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31, t4 = lane & 3;
  const int wg = blockIdx.x * wpc + warp;
  if (wg >= a.r) return;
  const int t = a.list ? a.list[wg] : wg;
  const int n = a.n[t];
  const int* I = a.I + a.I_off[t];
  const double* LiT = a.rec + a.L_off[t] + (int64_t)n * n;
  double* sY = smem + (size_t)warp * ldn * TW_LD;
  warp_stage32(sY, x, I, n);
  __syncwarp();
  auto epi = [&](int row, bool ok, double (&acc)[4][2]) {
    if (!ok) return;
    double* xr = x + (int64_t)__ldg(I + row) * 32 + 2 * t4;
#pragma unroll
    for (int y = 0; y < 4; ++y) *reinterpret_cast<double2*>(xr + 8 * y) = make_double2(acc[y][0], acc[y][1]);
  };
  if (up) warp_mm32<true>(LiT, n, n, n, 1, sY, epi);    // L^-1 = (L^-T)^T: lower
  else warp_mm32<false>(LiT, n, n, n, 3, sY, epi);      // L^-T: upper
}

// small separators (|g| <= 64, r > 0), 32 right-hand sides; records T (r x k~), X~^T (r x k~),
// L~^-T (k~ x k~):  up:   Y_r -= T^T Y_s ; Z = L~^-1 Y_r ; Y_s -= X~^T Z
//                    down: Y_r -= X~ Y_s  ; Z = L~^-T Y_r ; Y_s -= T Z      (x_R <- Z, x_S <- Y_s)
__global__ void __launch_bounds__(128) k_apply_skel_mma(ApplySkelArgs a, const int* list, int n, double* x, int up,
                                                        int ldrows) {
  extern __shared__ double smem[];
  const int wpc = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31, t4 = lane & 3;
  const int idx = blockIdx.x * wpc + warp;
  if (idx >= n) return;
  const int t = list[idx];
  const int r = a.r[t], kt = a.kt[t];
  const int* S = a.S + a.S_off[t];
  const int* R = a.R + a.R_off[t];
  const double* T = a.rec + a.T_off[t];                      // r x kt
  const double* PB = a.rec + a.P_off[t] + (int64_t)kt * kt;   // X~^T: r x kt
  const double* LiT = PB + (int64_t)r * kt;                  // L~^-T: kt x kt (upper)
  const int rp = (r + 3) & ~3, kp = (kt + 3) & ~3;
  double* sYs = smem + (size_t)warp * ldrows * TW_LD;
  double* sYr = sYs + (size_t)rp * TW_LD;
  double* sZ = sYr + (size_t)kp * TW_LD;
  warp_stage32(sYs, x, S, r);
  warp_stage32(sYr, x, R, kt);
  for (int i = kt; i < kp; ++i) sZ[i * TW_LD + lane] = 0.0;
  __syncwarp();
  const double* M1 = up ? T : PB;   // Y_r -= M1^T Y_s
  const double* M3 = up ? PB : T;   // Y_s -= M3 Z
  warp_mm32<true>(M1, kt, kt, r, 0, sYs, [&](int row, bool ok, double (&acc)[4][2]) {
    if (!ok) return;
    double* yr = sYr + row * TW_LD + 2 * t4;
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      yr[8 * y] -= acc[y][0];
      yr[8 * y + 1] -= acc[y][1];
    }
  });
  __syncwarp();
  auto epi2 = [&](int row, bool ok, double (&acc)[4][2]) {
    if (!ok) return;
    double* z = sZ + row * TW_LD + 2 * t4;
    double* xr = x + (int64_t)__ldg(R + row) * 32 + 2 * t4;
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      z[8 * y] = acc[y][0];
      z[8 * y + 1] = acc[y][1];
      *reinterpret_cast<double2*>(xr + 8 * y) = make_double2(acc[y][0], acc[y][1]);
    }
  };
  if (up) warp_mm32<true>(LiT, kt, kt, kt, 1, sYr, epi2);
  else warp_mm32<false>(LiT, kt, kt, kt, 3, sYr, epi2);
  __syncwarp();
  warp_mm32<false>(M3, kt, r, kt, 0, sZ, [&](int row, bool ok, double (&acc)[4][2]) {
    if (!ok) return;
    const double* ys = sYs + row * TW_LD + 2 * t4;
    double* xr = x + (int64_t)__ldg(S + row) * 32 + 2 * t4;
#pragma unroll
    for (int y = 0; y < 4; ++y)
      *reinterpret_cast<double2*>(xr + 8 * y) = make_double2(ys[8 * y] - acc[y][0], ys[8 * y + 1] - acc[y][1]);
  });
}

__global__ void __launch_bounds__(NT) k_apply_skel(ApplySkelArgs a, double* x, int k, int up) {
  extern __shared__ double smem[];
  const int t = a.list ? a.list[blockIdx.x] : blockIdx.x;
  const int r = a.r[t], kt = a.kt[t];
  if (kt == 0) return;
  const int* S = a.S + a.S_off[t];
  const int* R = a.R + a.R_off[t];
  const double* T = a.rec + a.T_off[t];
  const double* P = a.rec + a.P_off[t];
  const double* PB = P + (int64_t)kt * kt;
  double* Ys = a.work + a.work_off[t] * k;
  double* Yr = Ys + (int64_t)r * k;
  gather_rows(Ys, x, S, r, k);
  gather_rows(Yr, x, R, kt, k);
  __syncthreads();
  double* gsm = smem + GEMM_OFF;
  if (up) {
    if (r > 0) cta_gemm<true, false>(kt, k, r, -1.0, T, kt, Ys, k, 1.0, Yr, k, false, gsm);
    cta_trsm_left(P, kt, kt, Yr, k, k, false, smem);
    if (r > 0) cta_gemm<false, false>(r, k, kt, -1.0, PB, kt, Yr, k, 1.0, Ys, k, false, gsm);
  } else {
    if (r > 0) cta_gemm<true, false>(kt, k, r, -1.0, PB, kt, Ys, k, 1.0, Yr, k, false, gsm);
    cta_trsm_left(P, kt, kt, Yr, k, k, true, smem);
    if (r > 0) cta_gemm<false, false>(r, k, kt, -1.0, T, kt, Yr, k, 1.0, Ys, k, false, gsm);
  }
  scatter_rows(x, Ys, S, r, k);
  scatter_rows(x, Yr, R, kt, k);
}

// ---------------------------------------------------------------------------
// Krylov vector kernels (x is N x k row-major)
// ---------------------------------------------------------------------------
__global__ void k_spmv(const int64_t* rowptr, const int* col, const double* val, const double* x, double* y,
                       int64_t N, int k) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= N * k) return;
  const int64_t r = e / k;
  const int c = (int)(e % k);
  double s = 0.0;
  for (int64_t q = rowptr[r]; q < rowptr[r + 1]; ++q) s = __fma_rn(val[q], x[(int64_t)col[q] * k + c], s);
  y[e] = s;
}

// 32 right-hand sides: one warp per row, lane = right-hand side (no index division; the row's
// entries are warp-wide broadcasts, the x rows coalesced 256-byte reads). Same FMA order as k_spmv.
__global__ void __launch_bounds__(256) k_spmv32(const int64_t* __restrict__ rowptr, const int* __restrict__ col,
                                                const double* __restrict__ val, const double* x,
                                                double* y, int64_t N) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= N) return;
  const int64_t q0 = __ldg(rowptr + r), q1 = __ldg(rowptr + r + 1);
  double s = 0.0;
  for (int64_t q = q0; q < q1; ++q) s = __fma_rn(__ldg(val + q), x[(int64_t)__ldg(col + q) * 32 + lane], s);
  y[r * 32 + lane] = s;
}

// per-block partial column dot products: part[blk*k + c] = sum over the block's rows
__global__ void k_dot_part(const double* a, const double* b, int64_t N, int k, double* part) {
  extern __shared__ double sh[];
  const int c = threadIdx.x % k;           // blockDim.x is a multiple of k
  const int lanes = blockDim.x / k;
  const int row0 = threadIdx.x / k;
  double s = 0.0;
  for (int64_t r = (int64_t)blockIdx.x * lanes + row0; r < N; r += (int64_t)gridDim.x * lanes)
    s += a[r * k + c] * b[r * k + c];
  sh[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x < k) {
    double t = 0.0;
    for (int l = 0; l < lanes; ++l) t += sh[l * k + threadIdx.x];
    part[(int64_t)blockIdx.x * k + threadIdx.x] = t;
  }
}

// PCG update fused with the residual norm: x += alpha p ; r -= alpha q for active columns, and the
// per-block partial sums of r.r in the layout (and summation order) of k_dot_part, so the fused
// pass is bitwise identical to k_axpy, k_axpy, k_dot_part run one after the other
__global__ void k_pcg_update(double* x, const double* p, double* r, const double* q, const double* alpha,
                             const int* active, int64_t N, int k, double* part) {
  extern __shared__ double sh[];
  const int c = threadIdx.x % k;           // blockDim.x is a multiple of k
  const int lanes = blockDim.x / k;
  const int row0 = threadIdx.x / k;
  const bool on = active[c] != 0;
  const double al = alpha[c];
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * lanes + row0; i < N; i += (int64_t)gridDim.x * lanes) {
    const int64_t e = i * k + c;
    double rv = r[e];
    if (on) {
      x[e] += 1.0 * al * p[e];
      rv += -1.0 * al * q[e];
      r[e] = rv;
    }
    s += rv * rv;
  }
  sh[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x < k) {
    double t = 0.0;
    for (int l = 0; l < lanes; ++l) t += sh[l * k + threadIdx.x];
    part[(int64_t)blockIdx.x * k + threadIdx.x] = t;
  }
}

__global__ void k_dot_final(const double* part, int nblk, int k, double* out) {
  const int c = threadIdx.x;
  if (c >= k) return;
  double t = 0.0;
  for (int b = 0; b < nblk; ++b) t += part[(int64_t)b * k + c];
  out[c] = t;
}

// y[:,c] += s * coef[c] * x[:,c] for active columns
__global__ void k_axpy(double* y, const double* x, const double* coef, double s, const int* active, int64_t N,
                       int k) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= N * k) return;
  const int c = (int)(e % k);
  if (active && !active[c]) return;
  y[e] += s * coef[c] * x[e];
}

// p[:,c] = z[:,c] + coef[c] * p[:,c] for active columns
__global__ void k_xpby(double* p, const double* z, const double* coef, const int* active, int64_t N, int k) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= N * k) return;
  const int c = (int)(e % k);
  if (active && !active[c]) return;
  p[e] = z[e] + coef[c] * p[e];
}

// r[:,c] = b[:,c] - q[:,c] for active columns
__global__ void k_sub(double* r, const double* b, const double* q, const int* active, int64_t N, int k) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= N * k) return;
  const int c = (int)(e % k);
  if (active && !active[c]) return;
  r[e] = b[e] - q[e];
}

// out[c] = num[c] / den[c] for active, else 0
__global__ void k_ratio(const double* num, const double* den, const int* active, double* out, int k) {
  const int c = threadIdx.x;
  if (c >= k) return;
  out[c] = (active == nullptr || active[c]) ? num[c] / den[c] : 0.0;
}

// ---- PCG control on the device (one block; columns c < k) ----------------------------------
// ctl[0] = number of still-active columns, ctl[1] = first breakdown iteration (0 = none)
__global__ void k_pcg_init(const double* bn2, double* bn, int* active, double* relres, int* iters, int* conv,
                           int* ctl, int k) {
  if (threadIdx.x == 0) {
    ctl[0] = 0;
    ctl[1] = 0;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    const double b = sqrt(bn2[c]);
    bn[c] = b;
    iters[c] = 0;
    const bool a = b != 0.0;
    active[c] = a;
    relres[c] = a ? 1.0 : 0.0;
    conv[c] = a ? 0 : 1;
    if (a) atomicAdd(ctl, 1);
  }
}

__device__ __forceinline__ void pcg_flag_breakdown(int* ctl, int it) { atomicCAS(ctl + 1, 0, it); }

// alpha = rz / pq for active columns (0 otherwise)
__global__ void k_pcg_alpha(const double* rz, const double* pq, const int* active, double* alpha, int* ctl, int it,
                            int k) {
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    const double a = active[c] ? rz[c] / pq[c] : 0.0;
    if (!isfinite(a)) pcg_flag_breakdown(ctl, it);
    alpha[c] = a;
  }
}

// relative residuals, convergence, history row it-1 (every column, frozen ones keep their value)
__global__ void k_pcg_check(const double* rn2, const double* bn, int* active, double* relres, int* iters, int* conv,
                            double* hist, int it, double tol, int* ctl, int k) {
  if (threadIdx.x == 0) ctl[0] = 0;
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    if (active[c]) {
      const double rr = sqrt(rn2[c]) / bn[c];
      if (!isfinite(rr)) pcg_flag_breakdown(ctl, it);
      relres[c] = rr;
      iters[c] = it;
      if (rr <= tol) {
        active[c] = 0;
        conv[c] = 1;
      } else {
        atomicAdd(ctl, 1);
      }
    }
    if (hist) hist[(int64_t)(it - 1) * k + c] = relres[c];
  }
}

// beta = rzn / rz and rz <- rzn for active columns
__global__ void k_pcg_beta(const double* rzn, double* rz, const int* active, double* beta, int* ctl, int it, int k) {
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    if (active[c]) {
      const double b = rzn[c] / rz[c];
      if (!isfinite(b)) pcg_flag_breakdown(ctl, it);
      beta[c] = b;
      rz[c] = rzn[c];
    } else {
      beta[c] = 0.0;
    }
  }
}

// y = x - y (power iteration residual), y /= scale handled by k_scale
__global__ void k_xmy(double* y, const double* x, int64_t n) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) y[e] = x[e] - y[e];
}

__global__ void k_scale(double* y, const double* x, const double* nrm2, int64_t n) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) y[e] = x[e] / sqrt(nrm2[0]);
}

// ---------------------------------------------------------------------------
// Launch wrappers
// ---------------------------------------------------------------------------
std::atomic<long long> g_launches{0};
long long launch_count() { return g_launches.load(); }

static constexpr size_t SMEM_BYTES = (size_t)SMEM_DOUBLES * sizeof(double);

static inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }


// ---------------------------------------------------------------------------
// Streaming NT tile GEMM for the big cells (64 x 64 output tile per CTA, K streamed in
// 32-wide chunks through a 3-stage cp.async pipeline, DMMA m8n8k4, 2 CTAs per SM):
//  MODE 0: trailing update P[r, c] -= sum_{k0 <= k < k0+kw} P[r, k] P[c, k] for rows and
//          columns >= base = k0 + kw (tile (i, j) of that trailing block)
//  MODE 1: U = X^T X (X = rows n..n+b of P, K = n), lower tiles only, mirrored on write
// ---------------------------------------------------------------------------
constexpr int NTK = 32, NTLD = NTK + 4, NT_STAGES = 3;
constexpr int NT_STAGE = 2 * BT * NTLD;
constexpr size_t NT_SMEM = (size_t)NT_STAGES * NT_STAGE * sizeof(double);
constexpr int NT_CLD = BT + 1;   // C tile of the trailing update (MODE 0)
constexpr size_t NT_SMEM0 = (size_t)(2 * NT_STAGE + BT * NT_CLD) * sizeof(double);

// MODE 2 = MODE 0 without the C-tile prefetch: three K stages, C read (coalesced) in the epilogue
template <int MODE_>
__global__ void __launch_bounds__(NT, 2) k_big_nt(BigArgs a) {
  constexpr int MODE = MODE_ == 2 ? 0 : MODE_;
  constexpr bool CPRE = MODE_ == 0;
  extern __shared__ double smem[];
  const int c = a.w_cell[blockIdx.x], it = a.w_i[blockIdx.x], jt = a.w_j[blockIdx.x];
  const int n = a.n[c];
  double* P = a.P[c];
  int ar0, br0, kbeg, kend, Mv, Nv;
  if (MODE == 0) {
    const int base = a.k0 + a.kw;
    ar0 = base + BT * it;
    br0 = base + BT * jt;
    kbeg = a.k0;
    kend = a.k0 + a.kw;
    Mv = min(BT, a.rows[c] - ar0);
    Nv = min(BT, n - br0);
  } else {
    const int nb = n + a.b[c];
    ar0 = n + BT * it;
    br0 = n + BT * jt;
    kbeg = 0;
    kend = n;
    Mv = min(BT, nb - ar0);
    Nv = min(BT, nb - br0);
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 3, wn = warp >> 2, g = lane >> 2, t = lane & 3;
  const double* Ab = P + (int64_t)ar0 * n;
  const double* Bb = P + (int64_t)br0 * n;
  auto load = [&](int st, int kc) {
    double* sA = smem + st * NT_STAGE;
    double* sB = sA + BT * NTLD;
#pragma unroll
    for (int q = 0; q < (BT * NTK) / NT; ++q) {
      const int e = tid + q * NT, r = e / NTK, kk = e % NTK;
      const int gk = kc + kk;
      const bool okA = r < Mv && gk < kend, okB = r < Nv && gk < kend;
      cp_async8(sA + r * NTLD + kk, Ab + (okA ? (int64_t)r * n + gk : 0), okA);
      cp_async8(sB + r * NTLD + kk, Bb + (okB ? (int64_t)r * n + gk : 0), okB);
    }
    cp_async_commit();
  };
  // MODE 0 (trailing update C -= A B^T): the C tile is fetched into shared memory by cp.async
  // ahead of the K loop (2 stages, so two CTAs still fit per SM); its read-modify-write latency
  // no longer sits behind the last DMMA
  constexpr int STG = CPRE ? 2 : NT_STAGES;
  double* sC = smem + STG * NT_STAGE;
  if (CPRE) {
#pragma unroll
    for (int q = 0; q < (BT * BT) / NT; ++q) {
      const int e = tid + q * NT, r = e / BT, j = e % BT;
      const bool ok = r < Mv && j < Nv;
      cp_async8(sC + r * NT_CLD + j, P + (ok ? (int64_t)(ar0 + r) * n + br0 + j : 0), ok);
    }
    cp_async_commit();
  }
  double acc[2][4][2];
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  const int nch = (kend - kbeg + NTK - 1) / NTK;
#pragma unroll
  for (int st = 0; st < STG - 1; ++st)
    if (st < nch) load(st, kbeg + st * NTK);
  for (int ch = 0; ch < nch; ++ch) {
    if (ch + STG - 1 < nch) {
      load((ch + STG - 1) % STG, kbeg + (ch + STG - 1) * NTK);
      cp_async_wait<STG - 1>();
    } else if (STG == 3 && ch + 1 < nch) {
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* sA = smem + (ch % STG) * NT_STAGE;
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
  // epilogue through shared memory: the fragments land in the (padded) C tile, then whole rows
  // leave with coalesced stores (a warp writes 32 consecutive doubles of one row); the mirror
  // tile of U reads the staged tile by columns (conflict-free thanks to the padding)
  if (nch == 0) {   // (no K chunk: the C prefetch is still in flight)
    cp_async_wait<0>();
    __syncthreads();
  }
  double* sT = CPRE ? sC : smem;   // (otherwise the drained pipeline stages hold the tile)
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int z = 0; z < 2; ++z) {
        const int i = wm * 16 + x * 8 + g, j = wn * 32 + y * 8 + 2 * t + z;
        if (CPRE) sT[i * NT_CLD + j] -= acc[x][y][z];
        else sT[i * NT_CLD + j] = acc[x][y][z];
      }
  __syncthreads();
  if (MODE == 0) {
    for (int e = tid; e < BT * BT; e += NT) {
      const int i = e / BT, j = e % BT;
      if (i < Mv && j < Nv) {
        double* pc = P + (int64_t)(ar0 + i) * n + br0 + j;
        *pc = CPRE ? sT[i * NT_CLD + j] : *pc - sT[i * NT_CLD + j];
      }
    }
  } else {
    const int b = a.b[c];
    double* U = a.U[c];
    for (int e = tid; e < BT * BT; e += NT) {
      const int i = e / BT, j = e % BT;
      if (i < Mv && j < Nv) U[(int64_t)(BT * it + i) * b + BT * jt + j] = sT[i * NT_CLD + j];
    }
    if (it != jt)
      for (int e = tid; e < BT * BT; e += NT) {
        const int jj = e / BT, ii = e % BT;   // mirror row BT*jt + jj, column BT*it + ii
        if (ii < Mv && jj < Nv) U[(int64_t)(BT * jt + jj) * b + BT * it + ii] = sT[ii * NT_CLD + jj];
      }
  }
}

// ---------------------------------------------------------------------------
// 128 x 128 output tile variant of the streaming NT GEMM for the deep updates of the big cells
// (the KB-deep trailing updates and U = X^T X): one CTA per SM, 8 warps of 32 x 64, K streamed in
// 16-wide chunks through a 4-stage cp.async pipeline with one barrier per chunk. Twice the
// flops per byte fetched from L2 and half the cp.async / LDS instructions per DMMA of the
// 64 x 64 kernel. Tiles are counted in units of 128 from the same bases as k_big_nt.
//  MODE 0: P[r, c] -= sum_{k0 <= k < k0+kw} P[r, k] P[c, k]   (rows, columns >= k0 + kw)
//  MODE 1: U = X^T X (lower tiles; the mirror tile is written from the staged tile)
// Diagonal tiles skip the two warps whose 32 x 64 part lies strictly above the diagonal; identity
// rows (row n+b+i holds nonzeros in columns >= i only) start their K range at their first column.
// ---------------------------------------------------------------------------
constexpr int WT = 128, WTK = 16, WLD = WTK + 4, W_STAGES = 4;
constexpr int W_STAGE = 2 * WT * WLD;
constexpr int W_CLD = WT + 1;
constexpr size_t W_SMEM = (size_t)(W_STAGES * W_STAGE > WT * W_CLD ? W_STAGES * W_STAGE : WT * W_CLD) * sizeof(double);

template <int MODE>
__global__ void __launch_bounds__(NT, 1) k_big_wide(BigArgs a) {
  extern __shared__ double smem[];
  const int c = a.w_cell[blockIdx.x], it = a.w_i[blockIdx.x], jt = a.w_j[blockIdx.x];
  const int n = a.n[c];
  double* P = a.P[c];
  int ar0, br0, kbeg, kend, Mv, Nv;
  if (MODE == 0) {
    const int base = a.k0 + a.kw;
    ar0 = base + WT * it;
    br0 = base + WT * jt;
    kbeg = a.k0;
    kend = a.k0 + a.kw;
    Mv = min(WT, a.rows[c] - ar0);
    Nv = min(WT, n - br0);
    const int id0 = ar0 - (n + a.b[c]);   // first identity row of the tile (if >= 0)
    if (id0 > kbeg) kbeg = min(kend, id0 / WTK * WTK);
  } else {
    const int nb = n + a.b[c];
    ar0 = n + WT * it;
    br0 = n + WT * jt;
    kbeg = 0;
    kend = n;
    Mv = min(WT, nb - ar0);
    Nv = min(WT, nb - br0);
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 3, wn = warp >> 2, g = lane >> 2, t = lane & 3;
  const bool diag = it == jt;
  const bool skip = diag && wn == 1 && wm < 2;   // rows < 64, columns >= 64 of a diagonal tile
  const double* Ab = P + (int64_t)ar0 * n;
  const double* Bb = P + (int64_t)br0 * n;
  auto load = [&](int st, int kc) {
    double* sA = smem + st * W_STAGE;
    double* sB = sA + WT * WLD;
#pragma unroll
    for (int q = 0; q < (WT * WTK) / NT; ++q) {
      const int e = tid + q * NT, r = e / WTK, kk = e % WTK;
      const int gk = kc + kk;
      const bool okA = r < Mv && gk < kend, okB = r < Nv && gk < kend;
      cp_async8(sA + r * WLD + kk, Ab + (okA ? (int64_t)r * n + gk : 0), okA);
      cp_async8(sB + r * WLD + kk, Bb + (okB ? (int64_t)r * n + gk : 0), okB);
    }
  };
  double acc[4][8][2];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 8; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  const int nch = (kend - kbeg + WTK - 1) / WTK;
#pragma unroll
  for (int st = 0; st < W_STAGES - 1; ++st) {
    if (st < nch) load(st, kbeg + st * WTK);
    cp_async_commit();
  }
  if (MODE == 0) {   // C tile -> L2 (one 128-byte line per 16 columns of a row)
    for (int e = tid; e < WT * (WT / 16); e += NT) {
      const int i = e / (WT / 16), j = (e % (WT / 16)) * 16;
      if (i < Mv && j < Nv)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(P + (int64_t)(ar0 + i) * n + br0 + j));
    }
  }
  for (int ch = 0; ch < nch; ++ch) {
    cp_async_wait<W_STAGES - 2>();   // chunk ch has landed (one group is committed per iteration)
    __syncthreads();                 // ... for every thread; stage (ch - 1) % STAGES is drained
    if (ch + W_STAGES - 1 < nch) load((ch + W_STAGES - 1) % W_STAGES, kbeg + (ch + W_STAGES - 1) * WTK);
    cp_async_commit();
    if (skip) continue;
    const double* sA = smem + (ch % W_STAGES) * W_STAGE + (wm * 32 + g) * WLD + t;
    const double* sB = smem + (ch % W_STAGES) * W_STAGE + WT * WLD + (wn * 64 + g) * WLD + t;
#pragma unroll
    for (int ks = 0; ks < WTK; ks += 4) {
      double af[4], bf[8];
#pragma unroll
      for (int x = 0; x < 4; ++x) af[x] = sA[x * 8 * WLD + ks];
#pragma unroll
      for (int y = 0; y < 8; ++y) bf[y] = sB[y * 8 * WLD + ks];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 8; ++y) dmma(acc[x][y][0], acc[x][y][1], af[x], bf[y]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  // epilogue through shared memory (the drained pipeline stages): fragments -> padded tile,
  // then whole rows leave with coalesced accesses
  double* sT = smem;
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 8; ++y)
#pragma unroll
      for (int z = 0; z < 2; ++z) {
        const int i = wm * 32 + x * 8 + g, j = wn * 64 + y * 8 + 2 * t + z;
        sT[i * W_CLD + j] = acc[x][y][z];
      }
  __syncthreads();
  if (MODE == 0) {
    // read-modify-write of the C tile, 32 independent rows in flight per thread (the accumulator
    // registers are free by now); the tile was prefetched into L2 ahead of the K loop
    const int j = tid & (WT - 1), i0 = tid >> 7;   // NT = 256: two rows per pass
    if (j < Nv) {
      double* pc = P + (int64_t)ar0 * n + br0 + j;
      for (int ib = i0; ib < Mv; ib += 64) {
        double v[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          const int i = ib + 2 * u;
          v[u] = i < Mv ? pc[(int64_t)i * n] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          const int i = ib + 2 * u;
          if (i < Mv) pc[(int64_t)i * n] = v[u] - sT[i * W_CLD + j];
        }
      }
    }
  } else {
    const int b = a.b[c];
    double* U = a.U[c];
    for (int e = tid; e < WT * WT; e += NT) {
      const int i = e / WT, j = e % WT;
      if (i < Mv && j < Nv)
        U[(int64_t)(WT * it + i) * b + WT * jt + j] = (diag && j > i) ? sT[j * W_CLD + i] : sT[i * W_CLD + j];
    }
    if (!diag)
      for (int e = tid; e < WT * WT; e += NT) {
        const int jj = e / WT, ii = e % WT;   // mirror row WT*jt + jj, column WT*it + ii
        if (ii < Mv && jj < Nv) U[(int64_t)(WT * jt + jj) * b + WT * it + ii] = sT[ii * W_CLD + jj];
      }
  }
}

#include "gram_id.cuh"

void launch_ingest(const LevelDev& lv, const int* gid, const int* pos, const int64_t* rowptr, const int* col,
                   const double* val, int64_t N, cudaStream_t s) {
  if (N == 0) return;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  k_ingest<<<nblk(N, 256), 256, 0, s>>>(lv, gid, pos, rowptr, col, val, N);
}
__global__ void k_fill_int(int* p, int v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}
void launch_fill_int(int* p, int v, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  k_fill_int<<<std::min<int64_t>(nblk(n, 256), 148 * 8), 256, 0, s>>>(p, v, n);
}
void launch_group_pos(const LevelDev& lv, int* gid, int* pos, cudaStream_t s) {
  if (lv.G == 0) return;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  k_group_pos<<<nblk((int64_t)lv.G * 32, 256), 256, 0, s>>>(lv, gid, pos);
}
void launch_cell(const LevelDev& lv, const CellArgs& a, int count, DevStatus* st, cudaStream_t s) {
  if (count == 0) return;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  k_cell<<<count, NT, SMEM_BYTES, s>>>(lv, a, st);
}
void launch_schur(const LevelDev& lv, const SchurArgs& a, cudaStream_t s) {
  if (a.ntgt == 0) return;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const int ny = std::max(1, std::min(64, (148 * 8 + a.ntgt - 1) / a.ntgt));   // row split for few targets
  k_schur<<<dim3(a.ntgt, ny), NT, 0, s>>>(lv, a);
}
void launch_prec_build(const LevelDev& lv, const PrecArgs& a, const int* list, int nbig, cudaStream_t s) {
  if (!nbig) return;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  k_prec_build<<<nbig * 32, 256, 0, s>>>(lv, a, list, nbig, 32);
}
void launch_prec_factor(const LevelDev& lv, const PrecArgs& a, DevStatus* st, cudaStream_t s) {
  if (a.r == 0) return;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  k_prec_factor<<<a.r, NT, SMEM_BYTES, s>>>(lv, a, st);
}
void launch_prec_factor_warp(const LevelDev& lv, const PrecArgs& a, const int* list, int n, int kmax, DevStatus* st,
                             cudaStream_t s) {
  if (n == 0) return;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const size_t bytes = (size_t)8 * 2 * kmax * ((kmax + 1) | 1) * sizeof(double);
  if (bytes > 48 * 1024) cudaFuncSetAttribute(k_prec_factor_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  k_prec_factor_warp<<<(n + 7) / 8, 256, bytes, s>>>(lv, a, list, n, kmax, st);
}
void launch_prec_scale_warp(const LevelDev& lv, const PrecArgs& a, const int* list, int n, int ldmax, cudaStream_t s) {
  if (n == 0) return;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const size_t bytes = (size_t)8 * ldmax * ((ldmax + 1) | 1) * sizeof(double);
  if (bytes > 48 * 1024) cudaFuncSetAttribute(k_prec_scale_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  k_prec_scale_warp<<<(n + 7) / 8, 256, bytes, s>>>(lv, a, list, n, ldmax);
}
void launch_prec_scale(const LevelDev& lv, const PrecArgs& a, cudaStream_t s, bool gemm_only) {
  if (a.nscale == 0) return;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (gemm_only) {   // every block of the list has |g| |h| <= PREC_SCALE_T
    static bool init = false;
    if (!init) {
      cudaFuncSetAttribute(k_prec_scale_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)(SMEM_BYTES + PREC_SCALE_T * sizeof(double)));
      init = true;
    }
    k_prec_scale_gemm<<<a.nscale, NT, SMEM_BYTES + PREC_SCALE_T * sizeof(double), s>>>(lv, a);
    return;
  }
  k_prec_scale<<<a.nscale, NT, SMEM_BYTES + PREC_SCALE_T * sizeof(double), s>>>(lv, a);
}
static long long static_smem(const void* fn) {
  cudaFuncAttributes fa{};
  return cudaFuncGetAttributes(&fa, fn) == cudaSuccess ? (long long)fa.sharedSizeBytes : 16 * 1024;
}
template <int MINB>
static void launch_skel_id_dyn_t(const LevelDev& lv, const SkelArgs& a, const DynSched& ds, int64_t need_doubles,
                                 cudaStream_t s) {
  const int64_t cap_max = (227 * 1024 - static_smem((const void*)k_skel_id_dyn<MINB>) - 1024) / 8 - SMEM_DOUBLES;
  const int cap = (int)std::min<int64_t>(need_doubles, cap_max);
  const size_t bytes = SMEM_BYTES + (size_t)cap * sizeof(double);
  cudaFuncSetAttribute(k_skel_id_dyn<MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  int per_sm = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_skel_id_dyn<MINB>, NT, bytes);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = std::max(1, std::min(ds.count, std::max(per_sm, 1) * sms));
  k_skel_id_dyn<MINB><<<grid, NT, bytes, s>>>(lv, a, cap, ds);
}
void launch_skel_id_dyn(const LevelDev& lv, const SkelArgs& a, const DynSched& ds, int64_t need_doubles,
                        cudaStream_t s, int kmax) {
  if (ds.count == 0) return;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (kmax > 0 && kmax <= 12) launch_skel_id_dyn_t<3>(lv, a, ds, need_doubles, s);
  else launch_skel_id_dyn_t<2>(lv, a, ds, need_doubles, s);
}
void launch_skel_id(const LevelDev& lv, const SkelArgs& a, int count, int64_t need_doubles, cudaStream_t s) {
  if (count == 0) return;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const int64_t cap_max = (227 * 1024 - static_smem((const void*)k_skel_id) - 1024) / 8 - SMEM_DOUBLES;
  const int cap = (int)std::min<int64_t>(need_doubles, cap_max);
  const size_t bytes = SMEM_BYTES + (size_t)cap * sizeof(double);
  cudaFuncSetAttribute(k_skel_id, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  k_skel_id<<<count, NT, bytes, s>>>(lv, a, cap);
}
static size_t team_smem(int vcap, int kmax, int colcap) {
  return SMEM_BYTES + ((size_t)vcap + kmax + 1 + colcap) * sizeof(double);
}
int team_colcap(int vcap, int kmax) {
  // fill the CTA's shared memory (one team CTA per SM) with owned columns
  static long long static_bytes = -1;
  if (static_bytes < 0) {
    cudaFuncAttributes fa{};
    static_bytes = cudaFuncGetAttributes(&fa, k_skel_team) == cudaSuccess ? (long long)fa.sharedSizeBytes : 16 * 1024;
  }
  // 227 KB per block minus the static arrays and 1 KB the runtime reserves
  const long long avail = (227 * 1024 - static_bytes - 1024) / 8 - SMEM_DOUBLES - vcap - kmax - 1;
  return avail > 0 ? (int)avail : 0;
}
int team_blocks_per_sm(int vcap, int kmax, int colcap) {
  static size_t cached_bytes = 0;
  static int cached = 0;
  const size_t bytes = team_smem(vcap, kmax, colcap);
  if (bytes == cached_bytes) return cached;
  cudaFuncSetAttribute(k_skel_team, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_skel_team, NT, bytes);
  cached_bytes = bytes;
  cached = nb;
  return nb;
}
void launch_skel_team(const LevelDev& lv, const SkelArgs& a, const TeamArgs& t, int nblocks, cudaStream_t s) {
  if (nblocks == 0) return;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const size_t bytes = team_smem(t.vcap, t.kmax, t.colcap);
  cudaFuncSetAttribute(k_skel_team, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  LevelDev lv2 = lv;
  SkelArgs a2 = a;
  TeamArgs t2 = t;
  if (t.cluster > 0) {
    if (t.cluster > 8) cudaFuncSetAttribute(k_skel_team, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = t.cluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(nblocks);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = bytes;
    cfg.stream = s;
    cudaLaunchKernelEx(&cfg, k_skel_team, lv2, a2, t2);
    return;
  }
  void* args[] = {&lv2, &a2, &t2};
  cudaLaunchCooperativeKernel((void*)k_skel_team, dim3(nblocks), dim3(NT), args, bytes, s);
}
// co-resident clusters of `csize` team CTAs (0 if the cluster cannot be scheduled)
int team_max_clusters(int vcap, int kmax, int colcap, int csize) {
  const size_t bytes = team_smem(vcap, kmax, colcap);
  cudaFuncSetAttribute(k_skel_team, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (csize > 8) cudaFuncSetAttribute(k_skel_team, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = csize;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3(csize * 64);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = bytes;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, (void*)k_skel_team, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}
static constexpr size_t BIG_SMEM = 2 * BT * TLD * sizeof(double);
void launch_big_build(const LevelDev& lv, const CellArgs& ca, const int* big_cells, int nbig, cudaStream_t s) {
  if (!nbig) return;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const int chunks = 64;
  k_big_build<<<nbig * chunks, 256, 0, s>>>(lv, ca, big_cells, nbig, chunks);
}
void launch_big_step(const BigArgs& diag, const BigArgs& trsm, const BigArgs& upd, DevStatus* st, cudaStream_t s) {
  if (diag.nwork) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_big_diag<<<diag.nwork, NT, 0, s>>>(diag, st);
  }
  if (trsm.nwork) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_big_trsm<<<trsm.nwork, NT, BIG_SMEM, s>>>(trsm);
  }
  launch_big_nt(upd, 0, s);
}
static size_t band_smem(int nmax, int bmax, int w) {
  return ((size_t)nmax * (w + 1) + nmax + std::max<size_t>((size_t)bmax * 65, 8 * 32 * 17)) * sizeof(double);
}
bool band_cells_fit(int nmax, int bmax, int w) {
  const size_t bytes = band_smem(nmax, bmax, w);
  return w <= BAND_WMAX && nmax <= NT && bmax <= 64 && bytes <= 200 * 1024;
}
int64_t band_scratch_stride(int nmax, int w) { return (int64_t)nmax * (w + 2); }
void launch_cell_band(const LevelDev& lv, const CellArgs& ca, const int* list, int count, int nmax, int bmax, int w,
                      double* scratch, DevStatus* st, long long* prof, cudaStream_t s) {
  if (count == 0) return;
  const size_t bytes = band_smem(nmax, bmax, w);
  g_launches.fetch_add(2, std::memory_order_relaxed);
  const int64_t stride = band_scratch_stride(nmax, w);
  const int cb = (count + 7) / 8;
  if (w <= 15) {
    k_band_chol<15><<<cb, 256, 0, s>>>(lv, ca, list, count, w, scratch, stride, st);
    cudaFuncSetAttribute(k_cell_band<15>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    k_cell_band<15><<<count, NT, bytes, s>>>(lv, ca, list, w, st, prof, scratch, stride);
  } else {
    k_band_chol<BAND_WMAX><<<cb, 256, 0, s>>>(lv, ca, list, count, w, scratch, stride, st);
    cudaFuncSetAttribute(k_cell_band<BAND_WMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    k_cell_band<BAND_WMAX><<<count, NT, bytes, s>>>(lv, ca, list, w, st, prof, scratch, stride);
  }
}
void launch_band_check(const int64_t* rowptr, const int* col, const int* gid, const int* pos, const uint8_t* is_int,
                       int64_t N, int w, int* flag, cudaStream_t s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  k_band_check<<<nblk(N, 256), 256, 0, s>>>(rowptr, col, gid, pos, is_int, N, w, flag);
}
void launch_big_zero_upper(const BigArgs& a, cudaStream_t s) {
  if (!a.ncell) return;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const int chunks = 64;
  k_big_zero_upper<<<a.ncell * chunks, 256, 0, s>>>(a, chunks);
}
void launch_big_nt(const BigArgs& a, int mode, cudaStream_t s) {
  if (!a.nwork) return;
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(k_big_nt<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)NT_SMEM0);
    cudaFuncSetAttribute(k_big_nt<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)NT_SMEM);
    cudaFuncSetAttribute(k_big_nt<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)NT_SMEM);
    init = true;
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  static const bool no_cpre = getenv("PHIF_NT_NOCPRE") != nullptr;
  if (mode == 0 && no_cpre) k_big_nt<2><<<a.nwork, NT, NT_SMEM, s>>>(a);
  else if (mode == 0) k_big_nt<0><<<a.nwork, NT, NT_SMEM0, s>>>(a);
  else k_big_nt<1><<<a.nwork, NT, NT_SMEM, s>>>(a);
}
void launch_big_wide(const BigArgs& a, int mode, cudaStream_t s) {
  if (!a.nwork) return;
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(k_big_wide<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)W_SMEM);
    cudaFuncSetAttribute(k_big_wide<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)W_SMEM);
    init = true;
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (mode == 0) k_big_wide<0><<<a.nwork, NT, W_SMEM, s>>>(a);
  else k_big_wide<1><<<a.nwork, NT, W_SMEM, s>>>(a);
}
void launch_rgemm(const GemmDesc* desc, const int* w_desc, const int* w_tile, int nwork, int nrhs, cudaStream_t s,
                  int kmean) {
  if (!nwork) return;
  if (nrhs > 32) {
    launch_bgemm(desc, w_desc, w_tile, nwork, s);
    return;
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  // persistent CTAs, each streaming its items through the cross-item pipeline; the grid is a
  // multiple (PHIF_RG_WAVES) of the resident CTA count so the static striding balances
  static const int waves = [] {
    const char* e = getenv("PHIF_RG_WAVES");
    return e ? std::max(1, atoi(e)) : 2;
  }();
  static const int deep_at = [] {
    const char* e = getenv("PHIF_RG_DEEP");
    return e ? atoi(e) : 128;
  }();
  const bool deep = kmean >= deep_at;
  static const bool staged = getenv("PHIF_RG_SMEM") != nullptr;   // (measured on c5: 5.65 ms vs 5.37 ms for the fragment-load kernel, so off by default)
  if (deep && nrhs > 16 && staged) {
    static bool init = false;
    if (!init) {
      cudaFuncSetAttribute(k_rgemm_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RS_SMEM);
      init = true;
    }
    k_rgemm_smem<<<std::min(nwork, 148 * 16), NT, RS_SMEM, s>>>(desc, w_desc, w_tile, nwork);
  } else if (deep) {
    const int grid = std::min(nwork, 148 * 16);
    if (nrhs <= 8) k_rgemm_deep<1><<<grid, NT, 0, s>>>(desc, w_desc, w_tile, nwork);
    else if (nrhs <= 16) k_rgemm_deep<2><<<grid, NT, 0, s>>>(desc, w_desc, w_tile, nwork);
    else k_rgemm_deep<4><<<grid, NT, 0, s>>>(desc, w_desc, w_tile, nwork);
  } else {
    const int grid = std::min(nwork, 148 * 3 * waves);
    if (nrhs <= 8) k_rgemm<1, 32><<<grid, NT, 0, s>>>(desc, w_desc, w_tile, nwork, nrhs);
    else if (nrhs <= 16) k_rgemm<2, 32><<<grid, NT, 0, s>>>(desc, w_desc, w_tile, nwork, nrhs);
    else k_rgemm<4, 32><<<grid, NT, 0, s>>>(desc, w_desc, w_tile, nwork, nrhs);
  }
}
void launch_bgemm(const GemmDesc* desc, const int* w_desc, const int* w_tile, int nwork, cudaStream_t s) {
  if (!nwork) return;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const int grid = std::min(nwork, 148 * 16);
  k_bgemm<<<grid, NT, BG_SMEM, s>>>(desc, w_desc, w_tile, nwork);
}
void launch_rows(double* Y, double* x, const int* idx, const int64_t* seg_src, const int64_t* seg_dst,
                 const int* seg_len, int nseg, int k, bool to_x, cudaStream_t s) {
  if (!nseg) return;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const int grid = std::min((nseg + 7) / 8, 148 * 16);
  k_rows<<<grid, 256, 0, s>>>(Y, x, idx, seg_src, seg_dst, seg_len, nseg, k, to_x ? 1 : 0, 1);
}
void launch_skel_update(const LevelDev& lv, const SkelArgs& a, const int* list, int count, DevStatus* st,
                        cudaStream_t s) {
  if (count == 0) return;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  k_skel_update<<<count, NT, SMEM_BYTES, s>>>(lv, a, list, st);
}
void launch_skel_big_gather(const LevelDev& lv, const SkelArgs& a, const int* big, const int* idx,
                            const int64_t* idx_off, int nbig, cudaStream_t s) {
  if (!nbig) return;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  k_skel_big_gather<<<nbig * 64, 256, 0, s>>>(lv, a, big, idx, idx_off, nbig, 64);
}
void launch_skel_big_post(const LevelDev& lv, const SkelArgs& a, const int* big, const int* idx, const int64_t* idx_off,
                          const double* U, const int64_t* U_off, int nbig, cudaStream_t s) {
  if (!nbig) return;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  k_skel_big_post<<<nbig * 32, 256, 0, s>>>(lv, a, big, idx, idx_off, U, U_off, nbig, 32);
}
void launch_repack(const RepackArgs& a, cudaStream_t s) {
  if (a.nblk == 0) return;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const size_t bytes = (size_t)a.tab_cap * sizeof(RepackEnt);
  if (bytes > 48 * 1024) cudaFuncSetAttribute(k_repack, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  k_repack<<<a.nwork, NT, bytes, s>>>(a);
}
void launch_apply_cell(const ApplyCellArgs& a, double* x, int k, bool up, cudaStream_t s) {
  if (a.p == 0) return;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  k_apply_cell<<<a.p, NT, SMEM_BYTES, s>>>(a, x, k, up ? 1 : 0);
}
static bool apply_mma_enabled();
bool apply_cell_mma_fits(int nmax, int bmax, int k) { return k == 32 && nmax <= 32 && bmax <= 64 && apply_mma_enabled(); }
void launch_apply_cell_mma(const ApplyCellArgs& a, int nmax, int bmax, double* x, bool up, cudaStream_t s) {
  if (a.p == 0) return;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const int nrows = (nmax + 3) & ~3;
  const int ld = nrows + std::max(nrows, (bmax + 3) & ~3);
  const size_t per_warp = (size_t)ld * TW_LD * sizeof(double);
  const int wpc = 4;
  const size_t bytes = per_warp * wpc;
  static size_t set_bytes = 0;
  if (bytes > 48 * 1024 && bytes > set_bytes) {
    cudaFuncSetAttribute(k_apply_cell_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    set_bytes = bytes;
  }
  k_apply_cell_mma<<<(a.p + wpc - 1) / wpc, 32 * wpc, bytes, s>>>(a, x, up ? 1 : 0, nrows, ld);
}
void launch_apply_reduce(const int* dof, const int64_t* off, const int* rows, const double* wbuf, int nd, double* x,
                         int k, cudaStream_t s) {
  if (nd == 0) return;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  k_apply_reduce<<<nblk((int64_t)nd * k, 256), 256, 0, s>>>(dof, off, rows, wbuf, nd, x, k);
}
static bool apply_mma_enabled() {
  static const bool on = !getenv("PHIF_NO_APPLY_MMA");
  return on;
}
void launch_apply_prec(const ApplyPrecArgs& a, double* x, int k, bool up, cudaStream_t s) {
  if (a.r == 0) return;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (k == 32 && apply_mma_enabled()) {   // warp-level DMMA replay, rows staged in shared memory
    const int ldn = ((a.ldn > 0 ? a.ldn : 96) + 3) & ~3;
    const size_t per_warp = (size_t)ldn * TW_LD * sizeof(double);
    const int wpc = (int)std::max<size_t>(1, std::min<size_t>(8, (48 * 1024) / per_warp));
    const size_t bytes = per_warp * wpc;
    static size_t set_bytes = 0;
    if (bytes > 48 * 1024 && bytes > set_bytes) {
      cudaFuncSetAttribute(k_apply_prec_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
      set_bytes = bytes;
    }
    k_apply_prec_mma<<<(a.r + wpc - 1) / wpc, 32 * wpc, bytes, s>>>(a, x, up ? 1 : 0, ldn);
    return;
  }
  const int ldn = k <= 4 ? (a.ldn > 0 ? a.ldn : 96) : 0;   // shared-memory staging only for few RHS
  const size_t per_warp = (size_t)ldn * k * sizeof(double);
  const int wpc = ldn ? (int)std::max<size_t>(1, std::min<size_t>(8, (200 * 1024) / per_warp)) : 8;
  const size_t bytes = per_warp * wpc;
  static size_t set_bytes = 0;
  if (bytes > 48 * 1024 && bytes > set_bytes) {
    cudaFuncSetAttribute(k_apply_prec_tiny, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    set_bytes = bytes;
  }
  k_apply_prec_tiny<<<(a.r + wpc - 1) / wpc, 32 * wpc, bytes, s>>>(a, x, k, up ? 1 : 0, ldn);
}
void launch_fwd(const ApplyCellArgs* c, const ApplyPrecArgs* p, const ApplySkelArgs* sk, double* x, int k, bool up,
                cudaStream_t s) {
  if (c && c->p) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_fwd_cell<<<c->p, NT, 0, s>>>(*c, x, k, up ? 1 : 0);
  }
  if (p && p->r) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_fwd_prec<<<p->r, NT, 0, s>>>(*p, x, k, up ? 1 : 0);
  }
  if (sk && sk->nsk) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_fwd_skel<<<sk->nsk, NT, 0, s>>>(*sk, x, k, up ? 1 : 0);
  }
}
void launch_apply_skel_warp(const ApplySkelArgs& a, const int* list, int n, double* x, int k, bool up, int ldrows,
                            cudaStream_t s) {
  if (n == 0) return;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (k == 32 && apply_mma_enabled()) {
    const int ld = ldrows + 12;   // r, k~, k~ rows each padded to a multiple of 4
    const size_t per_warp = (size_t)ld * TW_LD * sizeof(double);
    const int wpc = (int)std::max<size_t>(1, std::min<size_t>(4, (64 * 1024) / per_warp));
    const size_t bytes = per_warp * wpc;
    static size_t set_bytes = 0;
    if (bytes > 48 * 1024 && bytes > set_bytes) {
      cudaFuncSetAttribute(k_apply_skel_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
      set_bytes = bytes;
    }
    k_apply_skel_mma<<<(n + wpc - 1) / wpc, 32 * wpc, bytes, s>>>(a, list, n, x, up ? 1 : 0, ld);
    return;
  }
  const size_t per_warp = (size_t)ldrows * k * sizeof(double);
  int wpc = (int)std::max<size_t>(1, std::min<size_t>(4, (200 * 1024) / per_warp));
  const size_t bytes = per_warp * wpc;
  static size_t set_bytes = 0;
  if (bytes > 48 * 1024 && bytes > set_bytes) {
    cudaFuncSetAttribute(k_apply_skel_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    set_bytes = bytes;
  }
  k_apply_skel_warp<<<(n + wpc - 1) / wpc, 32 * wpc, bytes, s>>>(a, list, n, x, k, up ? 1 : 0, ldrows);
}
void launch_apply_skel(const ApplySkelArgs& a, double* x, int k, bool up, cudaStream_t s) {
  if (a.nsk == 0) return;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  k_apply_skel<<<a.nsk, NT, SMEM_BYTES, s>>>(a, x, k, up ? 1 : 0);
}
void launch_spmv(const int64_t* rowptr, const int* col, const double* val, const double* x, double* y, int64_t N,
                 int k, cudaStream_t s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (k == 32) {
    k_spmv32<<<nblk(N * 32, 256), 256, 0, s>>>(rowptr, col, val, x, y, N);
    return;
  }
  k_spmv<<<nblk(N * k, 256), 256, 0, s>>>(rowptr, col, val, x, y, N, k);
}
int dot_part_blocks() { return 592; }
void launch_dot(const double* a, const double* b, int64_t N, int k, double* part, double* out, cudaStream_t s) {
  const int threads = (256 / k) * k;
  const int blocks = dot_part_blocks();
  g_launches.fetch_add(1, std::memory_order_relaxed);
  k_dot_part<<<blocks, threads, threads * sizeof(double), s>>>(a, b, N, k, part);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  k_dot_final<<<1, 32 * ((k + 31) / 32), 0, s>>>(part, blocks, k, out);
}
void launch_pcg_update(double* x, const double* p, double* r, const double* q, const double* alpha, const int* active,
                       int64_t N, int k, double* part, double* rn2, cudaStream_t s) {
  const int threads = (256 / k) * k;
  const int blocks = dot_part_blocks();
  g_launches.fetch_add(1, std::memory_order_relaxed);
  k_pcg_update<<<blocks, threads, threads * sizeof(double), s>>>(x, p, r, q, alpha, active, N, k, part);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  k_dot_final<<<1, 32 * ((k + 31) / 32), 0, s>>>(part, blocks, k, rn2);
}
void launch_axpy(double* y, const double* x, const double* coef, double sgn, const int* active, int64_t N, int k,
                 cudaStream_t s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  k_axpy<<<nblk(N * k, 256), 256, 0, s>>>(y, x, coef, sgn, active, N, k);
}
void launch_xpby(double* p, const double* z, const double* coef, const int* active, int64_t N, int k,
                 cudaStream_t s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  k_xpby<<<nblk(N * k, 256), 256, 0, s>>>(p, z, coef, active, N, k);
}
void launch_sub(double* r, const double* b, const double* q, const int* active, int64_t N, int k, cudaStream_t s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  k_sub<<<nblk(N * k, 256), 256, 0, s>>>(r, b, q, active, N, k);
}
static int ctl_threads(int k) { return std::min(1024, 32 * ((k + 31) / 32)); }
void launch_pcg_init(const double* bn2, double* bn, int* active, double* relres, int* iters, int* conv, int* ctl,
                     int k, cudaStream_t s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  k_pcg_init<<<1, ctl_threads(k), 0, s>>>(bn2, bn, active, relres, iters, conv, ctl, k);
}
void launch_pcg_alpha(const double* rz, const double* pq, const int* active, double* alpha, int* ctl, int it, int k,
                      cudaStream_t s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  k_pcg_alpha<<<1, ctl_threads(k), 0, s>>>(rz, pq, active, alpha, ctl, it, k);
}
void launch_pcg_check(const double* rn2, const double* bn, int* active, double* relres, int* iters, int* conv,
                      double* hist, int it, double tol, int* ctl, int k, cudaStream_t s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  k_pcg_check<<<1, ctl_threads(k), 0, s>>>(rn2, bn, active, relres, iters, conv, hist, it, tol, ctl, k);
}
void launch_pcg_beta(const double* rzn, double* rz, const int* active, double* beta, int* ctl, int it, int k,
                     cudaStream_t s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  k_pcg_beta<<<1, ctl_threads(k), 0, s>>>(rzn, rz, active, beta, ctl, it, k);
}
void launch_ratio(const double* num, const double* den, const int* active, double* out, int k, cudaStream_t s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  k_ratio<<<1, 32 * ((k + 31) / 32), 0, s>>>(num, den, active, out, k);
}
void launch_xmy(double* y, const double* x, int64_t n, cudaStream_t s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  k_xmy<<<nblk(n, 256), 256, 0, s>>>(y, x, n);
}
void launch_scale(double* y, const double* x, const double* nrm2, int64_t n, cudaStream_t s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  k_scale<<<nblk(n, 256), 256, 0, s>>>(y, x, nrm2, n);
}

// ---- Gram-path ID launches (gram_id.cuh) ----
static constexpr size_t GID_SMEM_CAP = 227 * 1024;
int gid_panel(int k) {
  static const int nb = getenv("PHIF_GID_NB") ? atoi(getenv("PHIF_GID_NB")) : 0;
  if (nb > 0) return std::max(4, std::min(nb, 16) & ~3);   // multiple of 4 (DMMA K steps)
  (void)k;
  return 16;   // measured: the widest panel the register blocking allows wins at every level
}
static int64_t gid_sreg(int k, int C) {
  // shared-memory Schur region: the packed share when it fits the CTA budget, else what is left
  // (columns beyond it spill to global memory); the back substitution stages in region + panel.
  // Even, so that the panel rows behind it stay 16-byte aligned (bulk copies).
  const int nb = gid_panel(k);
  const int64_t avail = ((int64_t)GID_SMEM_CAP - (int64_t)GidSmem::bytes(0, k, C, nb)) / (int64_t)sizeof(double);
  return std::min(avail, std::max<int64_t>(gid_pack0(k, C), std::max<int64_t>(0, (24 - nb) * (int64_t)k))) & ~(int64_t)1;
}
int gid_cluster(int kmax, bool* sg) {
  // smallest cluster whose per-CTA packed Schur share is at most `target` doubles
  static const int64_t target = getenv("PHIF_GID_PACK") ? atoll(getenv("PHIF_GID_PACK")) : 12288;
  static const int force_c = getenv("PHIF_GID_C") ? atoi(getenv("PHIF_GID_C")) : 0;
  int C = 16;
  if (force_c) {
    if (force_c != 1 && force_c != 2 && force_c != 4 && force_c != 8 && force_c != 16)
      throw std::runtime_error("PHIF_GID_C must be 1, 2, 4, 8 or 16");
    C = force_c;
  } else {
    for (int c : {1, 2, 4, 8, 16})
      if (gid_pack0(kmax, c) <= target) {
        C = c;
        break;
      }
  }
  *sg = gid_pack0(kmax, C) > gid_sreg(kmax, C);
  if (24 * (int64_t)kmax > gid_sreg(kmax, C) + (int64_t)gid_panel(kmax) * GidShape(kmax, C).ldp ||
      GidShape(kmax, C).nown0 > 128)
    throw std::runtime_error("gram ID: separator too large");
  return C;
}
// separators the Gram path can stage (back-substitution buffers in shared memory; at most 128
// owned columns per CTA)
bool gid_fits(int k) {
  const int64_t sreg = gid_sreg(k, 16);
  return 24 * (int64_t)k <= sreg + (int64_t)gid_panel(k) * GidShape(k, 16).ldp && GidShape(k, 16).nown0 <= 128;
}
int64_t gid_gbuf_doubles(int k, int C, bool sg, int S) {
  return (int64_t)S * k * k + (sg ? (int64_t)C * gid_pack0(k, C) : 0);
}
void launch_gid(const LevelDev& lv, const SkelArgs& a, const GramArgs& g, int kmax, bool sg, cudaStream_t s) {
  if (g.nitem == 0) return;
  LevelDev lv2 = lv;
  SkelArgs a2 = a;
  GramArgs g2 = g;
  g_launches.fetch_add(3, std::memory_order_relaxed);
  k_gid_count<<<g.nitem * g.P, NT, 0, s>>>(lv, a, g);
  k_gid_copy<<<g.nitem * g.P, NT, 0, s>>>(lv, a, g);
  static bool attr = false;
  if (!attr) {
    attr = true;
    cudaFuncSetAttribute(k_gid_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)NT_SMEM);
  }
  if (g.nwork) k_gid_gram<<<g.nwork, NT, NT_SMEM, s>>>(lv, a, g);
  int64_t sreg = gid_sreg(kmax, g.C);
  (void)sg;
  GramArgs g3 = g;
  g3.nb = gid_panel(kmax);
  const size_t bytes = GidSmem::bytes(sreg, kmax, g.C, g3.nb);
  // column slots per lane of the pivot-chain warp: 1, 2 or 4 by the owned columns per CTA
  const int nown0 = GidShape(kmax, g.C).nown0;
  void (*fn)(LevelDev, SkelArgs, GramArgs, int64_t) =
      nown0 <= 32 ? k_gid_cpqr<1> : (nown0 <= 64 ? k_gid_cpqr<2> : k_gid_cpqr<4>);
  cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = g.C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3(g.nitem * g.C);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = bytes;
  cfg.stream = s;
  cudaLaunchKernelEx(&cfg, fn, lv2, a2, g3, sreg);
}

// T of every Gram-path separator of the level in one launch (g.nitem items, g.CT CTAs each)
int64_t gid_T_cap(int kmax) {
  // staging doubles per CTA: what the CPQR kernel offered its back substitution (>= 24 kmax)
  return std::max<int64_t>(24 * (int64_t)kmax, std::min<int64_t>(25000, 64 * (int64_t)kmax));
}
void launch_gid_T(const LevelDev& lv, const SkelArgs& a, const GramArgs& g, int kmax, cudaStream_t s) {
  if (g.nitem == 0) return;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const size_t bytes = (size_t)g.tcap * sizeof(double) + 2 * (size_t)kmax * sizeof(int);
  cudaFuncSetAttribute(k_gid_T, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  k_gid_T<<<g.nitem * g.CT, NT, bytes, s>>>(lv, a, g);
}

void configure_kernels() {
  static bool done = false;
  if (done) return;
  done = true;
  const int bytes = (int)SMEM_BYTES;
  cudaFuncSetAttribute(k_cell, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_prec_factor, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_prec_scale, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       bytes + (int)(PREC_SCALE_T * sizeof(double)));
  cudaFuncSetAttribute(k_skel_id, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_skel_update, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_apply_cell, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_apply_prec, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_apply_skel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_big_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BIG_SMEM);
  cudaFuncSetAttribute(k_big_trsm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BIG_SMEM);
  cudaFuncSetAttribute(k_bgemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BG_SMEM);
}

}  // namespace phif
