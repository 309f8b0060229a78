// Microbenchmark of the team-QR block update (X -= V T^T V^T X, register-resident X slice):
// one CTA alone vs. every SM busy. nvcc -O3 -gencode arch=compute_100a,code=sm_100a qr_update_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int NT = 256;
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int mode>
__global__ void __launch_bounds__(NT, 1) k_upd(double* Wall, long long ldw, int ldp, int jb, int ncol, int reps,
                                               long long* cyc) {
  extern __shared__ double smem[];
  double* Vb = smem;
  __shared__ double s_Y[8][64], s_Z[64], Ts[64];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = 8, g8 = lane >> 2, t4 = lane & 3;
  double* W = Wall + (long long)blockIdx.x * ldw * 8;
  for (int e = tid; e < jb * ldp; e += NT) Vb[e] = 1e-3 * ((e * 7) % 13);
  if (tid < 64) Ts[tid] = (tid / 8 <= tid % 8) ? 0.1 : 0.0;
  __syncthreads();
  long long t0 = clock64(), tp1 = 0, tz = 0;
  for (int rep = 0; rep < reps; ++rep) {
    constexpr int QR_TPW = 40;
    const int ntile = (ldp + 7) >> 3;
    const int tpw = (ntile + nw - 1) / nw;
    const int t_lo = warp * tpw, t_hi = min(ntile, t_lo + tpw);
    const bool col_ok = g8 < ncol, va_ok = g8 < jb;
    double* Xc = W + (long long)min(g8, ncol - 1) * ldw;
    const double* Va = Vb + (long long)min(g8, jb - 1) * ldp;
    long long ta = clock64();
    double xr[QR_TPW][2];
    if constexpr (mode >= 2) {
      // sector layout: k-step z of a tile takes rows t4 + 4z (full 32-byte sectors per column)
#pragma unroll
      for (int u = 0; u < QR_TPW; ++u) {
        const int rr = (t_lo + u) * 8 + t4;
        const bool ok = t_lo + u < t_hi && col_ok;
        xr[u][0] = (ok && rr < ldp) ? __ldcg(Xc + rr) : 0.0;
        xr[u][1] = (ok && rr + 4 < ldp) ? __ldcg(Xc + rr + 4) : 0.0;
      }
    } else {
#pragma unroll
      for (int u = 0; u < QR_TPW; ++u) {
        const int rr = (t_lo + u) * 8 + 2 * t4;
        const bool ok = t_lo + u < t_hi && col_ok;
        xr[u][0] = (ok && rr < ldp) ? __ldcg(Xc + rr) : 0.0;
        xr[u][1] = (ok && rr + 1 < ldp) ? __ldcg(Xc + rr + 1) : 0.0;
      }
    }
    double c0 = 0.0, c1 = 0.0;
    if constexpr (mode == 1) {   // plain sum instead of the DMMA chain (isolates load time)
#pragma unroll
      for (int u = 0; u < QR_TPW; ++u) c0 += xr[u][0] + xr[u][1];
    } else if constexpr (mode >= 2) {
      double cc[4][2] = {};
#pragma unroll
      for (int u = 0; u < QR_TPW; ++u) {
        const int rr = (t_lo + u) * 8 + t4;
        if (t_lo + u < t_hi) {
          const double a0 = (va_ok && rr < ldp) ? Va[rr] : 0.0;
          const double a1 = (va_ok && rr + 4 < ldp) ? Va[rr + 4] : 0.0;
          dmma(cc[u & 3][0], cc[u & 3][1], a0, xr[u][0]);
          dmma(cc[u & 3][0], cc[u & 3][1], a1, xr[u][1]);
        }
      }
      c0 = (cc[0][0] + cc[1][0]) + (cc[2][0] + cc[3][0]);
      c1 = (cc[0][1] + cc[1][1]) + (cc[2][1] + cc[3][1]);
    } else {
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
    }
    s_Y[warp][g8 * 8 + 2 * t4] = c0;
    s_Y[warp][g8 * 8 + 2 * t4 + 1] = c1;
    __syncthreads();
    long long tb = clock64();
    tp1 += tb - ta;
    if constexpr (mode >= 2) {
      __shared__ double s_Yr[64];
      if (tid < 64) {
        double y = 0.0;
#pragma unroll
        for (int w2 = 0; w2 < 8; ++w2) y += s_Y[w2][tid];
        s_Yr[tid] = y;
      }
      __syncthreads();
      if (tid < 64) {
        const int bz = tid >> 3, col = tid & 7;
        double z = 0.0;
#pragma unroll
        for (int a = 0; a < 8; ++a)
          if (a <= bz) z += Ts[a * 8 + bz] * s_Yr[a * 8 + col];
        s_Z[tid] = z * 1e-6;
      }
    } else if (tid < 64) {
      const int bz = tid >> 3, col = tid & 7;
      double z = 0.0;
      for (int a = 0; a <= bz; ++a) {
        double y = 0.0;
        for (int w2 = 0; w2 < nw; ++w2) y += s_Y[w2][a * 8 + col];
        z += Ts[a * 8 + bz] * y;
      }
      s_Z[tid] = z * 1e-6;
    }
    __syncthreads();
    tz += clock64() - tb;
    const double za0 = -s_Z[t4 * 8 + g8], za1 = -s_Z[(t4 + 4) * 8 + g8];
    const double* V0 = Vb + (long long)min(t4, jb - 1) * ldp;
    const double* V1 = Vb + (long long)min(t4 + 4, jb - 1) * ldp;
    const bool b0_ok = t4 < jb, b1_ok = t4 + 4 < jb;
    const int nrow = (g8 & 1) ? (g8 >> 1) + 4 : (g8 >> 1);   // N index g -> row of the tile
#pragma unroll
    for (int u = 0; u < QR_TPW; ++u) {
      if (t_lo + u < t_hi) {
        const int rv = (t_lo + u) * 8 + (mode >= 2 ? nrow : g8);
        const double vb0 = (b0_ok && rv < ldp) ? V0[rv] : 0.0;
        const double vb1 = (b1_ok && rv < ldp) ? V1[rv] : 0.0;
        dmma(xr[u][0], xr[u][1], za0, vb0);
        dmma(xr[u][0], xr[u][1], za1, vb1);
        if constexpr (mode >= 2) {
          const int rr = (t_lo + u) * 8 + t4;
          if (col_ok) {
            if (rr < ldp) __stcg(Xc + rr, xr[u][0]);
            if (rr + 4 < ldp) __stcg(Xc + rr + 4, xr[u][1]);
          }
        } else {
          const int rr = (t_lo + u) * 8 + 2 * t4;
          if (col_ok) {
            if (rr < ldp) __stcg(Xc + rr, xr[u][0]);
            if (rr + 1 < ldp) __stcg(Xc + rr + 1, xr[u][1]);
          }
        }
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) {
    cyc[3 * blockIdx.x] = (t1 - t0) / reps;
    cyc[3 * blockIdx.x + 1] = tp1 / reps;
    cyc[3 * blockIdx.x + 2] = tz / reps;
  }
}
int main() {
  const int ldp = 2373;
  const long long ldw = 2400;
  double* W;
  long long* cyc;
  cudaMalloc(&W, 148LL * ldw * 8 * 8);
  cudaMemset(W, 0, 148LL * ldw * 8 * 8);
  cudaMallocManaged(&cyc, 3 * 148 * sizeof(long long));
  const size_t smem = 8 * ldp * 8;
  cudaFuncSetAttribute(k_upd<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_upd<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int mode : {0, 2})
    for (int jb : {4, 8})
      for (int grid : {1, 148}) {
        if (mode == 2) {
          k_upd<2><<<grid, NT, smem>>>(W, ldw, ldp, jb, jb, 2, cyc);
          k_upd<2><<<grid, NT, smem>>>(W, ldw, ldp, jb, jb, 50, cyc);
        } else {
          k_upd<0><<<grid, NT, smem>>>(W, ldw, ldp, jb, jb, 2, cyc);
          k_upd<0><<<grid, NT, smem>>>(W, ldw, ldp, jb, jb, 50, cyc);
        }
        cudaError_t e = cudaDeviceSynchronize();
        if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        printf("mode %s jb=ncol=%d grid=%3d: %lld cycles/update (pass1 %lld, Z %lld)\n", mode == 2 ? "new " : "old ", jb, grid,
               cyc[0], cyc[1], cyc[2]);
      }
  return 0;
}
