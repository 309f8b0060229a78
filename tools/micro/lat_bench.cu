// Dependent-latency microbenchmarks (cycles per op, one warp / one CTA): DFMA, sqrt, 1/x, rsqrt,
// shuffle-based argmax, redux-based argmax, __syncthreads, LDS chain.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o lat_bench lat_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
#define N 512
__global__ void k(double* out, long long* cyc, double x0) {
  __shared__ double sm[1024];
  __shared__ int si[1024];
  const int tid = threadIdx.x, lane = tid & 31;
  double x = x0 + tid * 1e-9;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = __fma_rn(x, 1.0000001, 1e-12);
  t1 = clock64();
  if (tid == 0) cyc[0] = t1 - t0;
  // sqrt chain
  t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N; ++i) x = sqrt(x + 2.0);
  t1 = clock64();
  if (tid == 0) cyc[1] = t1 - t0;
  // div chain
  t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N; ++i) x = 1.0 / (x + 0.5);
  t1 = clock64();
  if (tid == 0) cyc[2] = t1 - t0;
  // rsqrt chain
  t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N; ++i) x = rsqrt(x + 2.0);
  t1 = clock64();
  if (tid == 0) cyc[3] = t1 - t0;
  // shuffle argmax (double value + int index), 5 levels
  int idx = tid;
  t0 = clock64();
  for (int i = 0; i < N; ++i) {
    double v = x + lane * 1e-3 * (i & 3);
    int bi = idx;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double y = __shfl_xor_sync(0xffffffffu, v, o);
      const int yi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (y > v || (y == v && yi < bi)) { v = y; bi = yi; }
    }
    x = v; idx = bi + lane;
  }
  t1 = clock64();
  if (tid == 0) cyc[4] = t1 - t0;
  // redux argmax: hi word max, lo word max among ties, min index among ties
  t0 = clock64();
  for (int i = 0; i < N; ++i) {
    const double v = x + lane * 1e-3 * (i & 3);
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    const unsigned hi = (unsigned)(b >> 32), lo = (unsigned)b;
    const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
    const unsigned mi = __reduce_min_sync(0xffffffffu, (hi == mh && lo == ml) ? (unsigned)idx : 0xffffffffu);
    x = __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
    idx = (int)mi + lane;
  }
  t1 = clock64();
  if (tid == 0) cyc[5] = t1 - t0;
  // __syncthreads chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) __syncthreads();
  t1 = clock64();
  if (tid == 0) cyc[6] = t1 - t0;
  // LDS pointer chase
  si[tid] = (tid * 7 + 1) & 1023;
  si[tid + 256] = (tid * 5 + 3) & 1023; si[tid + 512] = (tid * 3 + 7) & 1023; si[tid + 768] = (tid + 11) & 1023;
  __syncthreads();
  int p = tid;
  t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < N; ++i) p = si[p];
  t1 = clock64();
  if (tid == 0) cyc[7] = t1 - t0;
  // STS -> barrier -> LDS round trip (publish/consume)
  t0 = clock64();
  for (int i = 0; i < N; ++i) {
    if (tid == (i & 255)) sm[i & 1] = x;
    __syncthreads();
    x += sm[i & 1] * 1e-9;
  }
  t1 = clock64();
  if (tid == 0) cyc[8] = t1 - t0;
  // DSETP/fmax chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = fmax(x, x0 + i);
  t1 = clock64();
  if (tid == 0) cyc[9] = t1 - t0;
  out[tid] = x + p + idx;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 16 * 8);
  const char* names[] = {"dfma", "sqrt", "div", "rsqrt", "shfl-argmax", "redux-argmax", "syncthreads", "lds-chase", "sts-bar-lds", "fmax"};
  for (int nt : {32, 256}) {
    k<<<1, nt>>>(out, cyc, 1.5);
    cudaDeviceSynchronize();
    k<<<1, nt>>>(out, cyc, 1.5);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("error\n"); return 1; }
    printf("threads %d:", nt);
    for (int i = 0; i < 10; ++i) printf(" %s %.1f", names[i], (double)cyc[i] / N);
    printf("\n");
  }
  return 0;
}
