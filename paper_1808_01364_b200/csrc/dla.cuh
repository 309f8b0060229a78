// CTA-cooperative FP64 dense linear algebra for sm_100a.
//
// Every routine here is called by ALL threads of a CTA (blockDim.x == NT) and
// works on row-major matrices in global memory (M(i,j) = p[i*ld + j]), staging
// tiles through shared memory. They are the building blocks of the batched
// stage kernels (one CTA per cell / group / block). The GEMM core uses the
// FP64 tensor-core MMA (mma.sync m8n8k4 .f64 -> DMMA on sm_100a; tcgen05 has
// no f64 kind).
//
// Semantics follow LAPACK as called by the reference (kernels.py:23-119):
//  * potrf: lower, unpivoted, natural order; first pivot <= 0 (or NaN) is
//    reported 0-based like kernels.py:32.
//  * trsm: forward/back substitution with the lower factor.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#ifndef PHIF_NT
#define PHIF_NT 256
#endif

namespace phif {

constexpr int NT = PHIF_NT;
constexpr int NB = 32;          // panel width of the blocked factorizations

__device__ __forceinline__ double ld_a(const double* p) { return __ldg(p); }

// ---------------------------------------------------------------------------
// Warp / CTA reductions
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// CTA-wide sum; `red` is a shared scratch of >= NT/32 doubles. All threads get the result.
__device__ __forceinline__ double cta_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (w == 0) {
    s = (l < NT / 32) ? red[l] : 0.0;
    s = warp_sum(s);
    if (l == 0) red[0] = s;
  }
  __syncthreads();
  s = red[0];
  __syncthreads();
  return s;
}

// ---------------------------------------------------------------------------
// DMMA m8n8k4 (A row-major 8x4, B col-major 4x8, C 8x8 f64)
// lane: g = lane>>2, t = lane&3 ; a = A[g][t] ; b = B[t][g] ; c = C[g][2t+{0,1}]
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// C[M x N] = beta*C + alpha * op(A) * op(B), op(A) is M x K, op(B) is K x N.
//   TA=false: A(i,k) = A[i*lda+k]   TA=true: A(i,k) = A[k*lda+i]
//   TB=false: B(k,j) = B[k*ldb+j]   TB=true: B(k,j) = B[j*ldb+k]
// lower=true: only output tiles intersecting the lower triangle (i >= j) are
// computed (tiles strictly above are skipped; diagonal tiles written fully).
// smem: needs gemm_smem_doubles() doubles.
// ---------------------------------------------------------------------------
constexpr int GBM = 64, GBN = 64, GBK = 16, GLD = 68;   // GLD % 16 == 4: conflict-free fragments
__host__ __device__ constexpr int gemm_smem_doubles() { return 2 * GBK * GLD; }

template <bool TA, bool TB>
__device__ void cta_gemm(int M, int N, int K, double alpha, const double* __restrict__ A, int lda,
                         const double* __restrict__ B, int ldb, double beta, double* C, int ldc,
                         bool lower, double* smem) {
  if (M <= 0 || N <= 0) return;
  double* sA = smem;              // [GBK][GLD]  sA[k][i]
  double* sB = smem + GBK * GLD;  // [GBK][GLD]  sB[k][j]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 3, wn = warp >> 2;   // 4 x 2 warps, warp tile 16 x 32
  const int g = lane >> 2, t = lane & 3;
  const int tiles_m = (M + GBM - 1) / GBM, tiles_n = (N + GBN - 1) / GBN;
  for (int tile = 0; tile < tiles_m * tiles_n; ++tile) {
    const int tm = tile / tiles_n, tn = tile % tiles_n;
    const int i0 = tm * GBM, j0 = tn * GBN;
    if (lower && j0 > i0 + GBM - 1) continue;
    double acc[2][4][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    if (K > 0) {
      for (int k0 = 0; k0 < K; k0 += GBK) {
        __syncthreads();
        // load A tile: 64 x 16
        for (int e = tid; e < GBM * GBK; e += NT) {
          int ii, kk;
          if (TA) { kk = e / GBM; ii = e % GBM; } else { ii = e / GBK; kk = e % GBK; }
          const int gi = i0 + ii, gk = k0 + kk;
          double v = 0.0;
          if (gi < M && gk < K) v = TA ? A[(size_t)gk * lda + gi] : A[(size_t)gi * lda + gk];
          sA[kk * GLD + ii] = v;
        }
        for (int e = tid; e < GBN * GBK; e += NT) {
          int jj, kk;
          if (TB) { jj = e / GBK; kk = e % GBK; } else { kk = e / GBN; jj = e % GBN; }
          const int gj = j0 + jj, gk = k0 + kk;
          double v = 0.0;
          if (gj < N && gk < K) v = TB ? B[(size_t)gj * ldb + gk] : B[(size_t)gk * ldb + gj];
          sB[kk * GLD + jj] = v;
        }
        __syncthreads();
#pragma unroll
        for (int ks = 0; ks < GBK; ks += 4) {
          double af[2], bf[4];
#pragma unroll
          for (int a = 0; a < 2; ++a) af[a] = sA[(ks + t) * GLD + wm * 16 + a * 8 + g];
#pragma unroll
          for (int b = 0; b < 4; ++b) bf[b] = sB[(ks + t) * GLD + wn * 32 + b * 8 + g];
#pragma unroll
          for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        }
      }
    }
    // epilogue
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int gi = i0 + wm * 16 + a * 8 + g;
          const int gj = j0 + wn * 32 + b * 8 + 2 * t + c;
          if (gi < M && gj < N) {
            double* p = C + (size_t)gi * ldc + gj;
            *p = (beta == 0.0 ? 0.0 : beta * *p) + alpha * acc[a][b][c];
          }
        }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Factor a kb x kb (kb <= NB) SPD tile held in smem D[NB][NB+1] (lower, in place).
// Returns -1 on success, else the local 0-based failing pivot (all threads).
// ---------------------------------------------------------------------------
constexpr int DLD = NB + 1;
__device__ int cta_potrf_tile(double* D, int kb, int* sflag) {
  const int tid = threadIdx.x;
  if (tid == 0) *sflag = -1;
  __syncthreads();
  for (int j = 0; j < kb; ++j) {
    const double d = D[j * DLD + j];
    if (!(d > 0.0)) {           // pivot <= 0 or NaN: dpotrf info = j+1
      if (tid == 0) *sflag = j;
      __syncthreads();
      return *sflag;
    }
    const double ljj = sqrt(d);
    __syncthreads();
    if (tid == 0) D[j * DLD + j] = ljj;
    for (int i = j + 1 + tid; i < kb; i += NT) D[i * DLD + j] /= ljj;
    __syncthreads();
    const int m = kb - j - 1;
    for (int e = tid; e < m * m; e += NT) {
      const int i = j + 1 + e / m, k = j + 1 + e % m;
      if (k <= i) D[i * DLD + k] -= D[i * DLD + j] * D[k * DLD + j];
    }
    __syncthreads();
  }
  return -1;
}

// ---------------------------------------------------------------------------
// Partial Cholesky of a tall row-major panel P (nrows x n, nrows >= n):
//   L = chol(P[0:n,0:n]) in place (strict upper zeroed), rows n..nrows-1 become
//   P[n:,:] L^-T. Right-looking, NB-wide panels, DMMA trailing update.
// Returns -1 or the 0-based failing pivot. smem: >= potrf_smem_doubles().
// ---------------------------------------------------------------------------
// shared-memory layout used by every routine: [0, NB*DLD) diag tile, flags at
// NB*DLD+32, [NB*DLD+64, +gemm_smem_doubles()) GEMM staging, then RED_OFF.. reductions
constexpr int GEMM_OFF = NB * DLD + 64;
constexpr int RED_OFF = GEMM_OFF + 2 * GBK * GLD;
constexpr int SMEM_DOUBLES = RED_OFF + 64;
__host__ __device__ constexpr int potrf_smem_doubles() { return SMEM_DOUBLES; }

__device__ int cta_potrf_panel(double* P, int nrows, int n, int ld, double* smem) {
  double* D = smem;                                   // NB x DLD diag tile
  int* sflag = reinterpret_cast<int*>(smem + NB * DLD + 32);
  double* gsm = smem + GEMM_OFF;                      // gemm scratch (after diag tile)
  const int tid = threadIdx.x;
  for (int k0 = 0; k0 < n; k0 += NB) {
    const int kb = min(NB, n - k0);
    __syncthreads();
    for (int e = tid; e < NB * NB; e += NT) {
      const int i = e / NB, j = e % NB;
      D[i * DLD + j] = (i < kb && j <= i) ? P[(size_t)(k0 + i) * ld + k0 + j] : 0.0;
    }
    __syncthreads();
    const int bad = cta_potrf_tile(D, kb, sflag);
    if (bad >= 0) return k0 + bad;
    for (int e = tid; e < kb * kb; e += NT) {
      const int i = e / kb, j = e % kb;
      P[(size_t)(k0 + i) * ld + k0 + j] = (j <= i) ? D[i * DLD + j] : 0.0;
    }
    // TRSM rows below: x * D^T = p  (thread per row)
    for (int r = k0 + kb + tid; r < nrows; r += NT) {
      double x[NB];
      double* pr = P + (size_t)r * ld + k0;
#pragma unroll
      for (int j = 0; j < NB; ++j) x[j] = (j < kb) ? pr[j] : 0.0;
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        if (j < kb) {
          double s = x[j];
#pragma unroll
          for (int i = 0; i < NB; ++i)
            if (i < j) s -= x[i] * D[j * DLD + i];
          x[j] = s / D[j * DLD + j];
        }
      }
#pragma unroll
      for (int j = 0; j < NB; ++j)
        if (j < kb) pr[j] = x[j];
    }
    __syncthreads();
    // zero the strict upper part of this column block inside the square part
    for (int e = tid; e < kb * k0; e += NT) {
      const int i = e / k0, j = e % k0;
      P[(size_t)j * ld + k0 + i] = 0.0;
    }
    // trailing update: P[k0+kb:, k0+kb:n] -= P[k0+kb:, k0:k0+kb] * P[k0+kb:n, k0:k0+kb]^T
    const int r0 = k0 + kb;
    if (r0 < n) {
      // square part (lower only) and the tall part below
      cta_gemm<false, true>(n - r0, n - r0, kb, -1.0, P + (size_t)r0 * ld + k0, ld,
                            P + (size_t)r0 * ld + k0, ld, 1.0, P + (size_t)r0 * ld + r0, ld, true, gsm);
      if (nrows > n)
        cta_gemm<false, true>(nrows - n, n - r0, kb, -1.0, P + (size_t)n * ld + k0, ld,
                              P + (size_t)r0 * ld + k0, ld, 1.0, P + (size_t)n * ld + r0, ld, false, gsm);
    }
  }
  __syncthreads();
  return -1;
}

// ---------------------------------------------------------------------------
// Y = L^-1 Y (trans=false) or Y = L^-T Y (trans=true); L n x n lower (ldl),
// Y n x m row-major (ldy). Blocked: NB diag tile in smem, DMMA updates.
// smem: potrf_smem_doubles().
// ---------------------------------------------------------------------------
__device__ void cta_trsm_left(const double* L, int n, int ldl, double* Y, int m, int ldy, bool trans,
                              double* smem) {
  if (n <= 0 || m <= 0) return;
  double* D = smem;
  double* gsm = smem + GEMM_OFF;
  const int tid = threadIdx.x;
  const int nblk = (n + NB - 1) / NB;
  for (int bi = 0; bi < nblk; ++bi) {
    const int blk = trans ? (nblk - 1 - bi) : bi;
    const int k0 = blk * NB, kb = min(NB, n - k0);
    __syncthreads();
    for (int e = tid; e < NB * NB; e += NT) {
      const int i = e / NB, j = e % NB;
      D[i * DLD + j] = (i < kb && j <= i) ? L[(size_t)(k0 + i) * ldl + k0 + j] : 0.0;
    }
    __syncthreads();
    // solve the kb rows of Y in place, one column of Y per thread
    for (int c = tid; c < m; c += NT) {
      double x[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) x[j] = (j < kb) ? Y[(size_t)(k0 + j) * ldy + c] : 0.0;
      if (!trans) {
#pragma unroll
        for (int j = 0; j < NB; ++j)
          if (j < kb) {
            double s = x[j];
#pragma unroll
            for (int i = 0; i < NB; ++i)
              if (i < j) s -= D[j * DLD + i] * x[i];
            x[j] = s / D[j * DLD + j];
          }
      } else {
#pragma unroll
        for (int jj = NB - 1; jj >= 0; --jj)
          if (jj < kb) {
            double s = x[jj];
#pragma unroll
            for (int i = 0; i < NB; ++i)
              if (i > jj && i < kb) s -= D[i * DLD + jj] * x[i];
            x[jj] = s / D[jj * DLD + jj];
          }
      }
#pragma unroll
      for (int j = 0; j < NB; ++j)
        if (j < kb) Y[(size_t)(k0 + j) * ldy + c] = x[j];
    }
    __syncthreads();
    if (!trans) {
      // Y[k0+kb:n] -= L[k0+kb:n, k0:k0+kb] * Y[k0:k0+kb]
      const int r0 = k0 + kb;
      if (r0 < n)
        cta_gemm<false, false>(n - r0, m, kb, -1.0, L + (size_t)r0 * ldl + k0, ldl, Y + (size_t)k0 * ldy, ldy,
                               1.0, Y + (size_t)r0 * ldy, ldy, false, gsm);
    } else {
      // Y[0:k0] -= L[k0:k0+kb, 0:k0]^T * Y[k0:k0+kb]
      if (k0 > 0)
        cta_gemm<true, false>(k0, m, kb, -1.0, L + (size_t)k0 * ldl, ldl, Y + (size_t)k0 * ldy, ldy, 1.0, Y,
                              ldy, false, gsm);
    }
  }
  __syncthreads();
}

// Y = Y L^-T  (Y m x n row-major): each row y solves y L^T = p, i.e. (L y^T = p^T).
// Implemented as the transpose-free dual of cta_trsm_left on rows.
__device__ void cta_trsm_right_lt(const double* L, int n, int ldl, double* Y, int m, int ldy, double* smem) {
  if (n <= 0 || m <= 0) return;
  double* D = smem;
  double* gsm = smem + GEMM_OFF;
  const int tid = threadIdx.x;
  for (int k0 = 0; k0 < n; k0 += NB) {
    const int kb = min(NB, n - k0);
    __syncthreads();
    for (int e = tid; e < NB * NB; e += NT) {
      const int i = e / NB, j = e % NB;
      D[i * DLD + j] = (i < kb && j <= i) ? L[(size_t)(k0 + i) * ldl + k0 + j] : 0.0;
    }
    __syncthreads();
    for (int r = tid; r < m; r += NT) {
      double x[NB];
      double* pr = Y + (size_t)r * ldy + k0;
#pragma unroll
      for (int j = 0; j < NB; ++j) x[j] = (j < kb) ? pr[j] : 0.0;
#pragma unroll
      for (int j = 0; j < NB; ++j)
        if (j < kb) {
          double s = x[j];
#pragma unroll
          for (int i = 0; i < NB; ++i)
            if (i < j) s -= x[i] * D[j * DLD + i];
          x[j] = s / D[j * DLD + j];
        }
#pragma unroll
      for (int j = 0; j < NB; ++j)
        if (j < kb) pr[j] = x[j];
    }
    __syncthreads();
    const int c0 = k0 + kb;
    if (c0 < n)   // Y[:, c0:n] -= Y[:, k0:k0+kb] * L[c0:n, k0:k0+kb]^T
      cta_gemm<false, true>(m, n - c0, kb, -1.0, Y + k0, ldy, L + (size_t)c0 * ldl + k0, ldl, 1.0, Y + c0, ldy,
                            false, gsm);
  }
  __syncthreads();
}

}  // namespace phif
