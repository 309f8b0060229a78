// Microbenchmark: DMMA m8n8k4 latency/throughput and batched L2 load latency on one SM.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a dmma_bench.cu -o dmma_bench
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k_chain(double* out, long long* cyc, int iters) {
  double c0[CH], c1[CH];
  for (int i = 0; i < CH; ++i) c0[i] = c1[i] = threadIdx.x;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) dmma(c0[i], c1[i], a, b);
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < CH; ++i) s += c0[i] + c1[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void k_ffma(double* out, long long* cyc, int iters) {
  double c[8];
  for (int i = 0; i < 8; ++i) c[i] = threadIdx.x;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fma(c[i], a, b);
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int NL>
__global__ void k_loads(const double* src, double* out, long long* cyc, int stride) {
  __syncthreads();
  long long t0 = clock64();
  double v[NL];
#pragma unroll
  for (int u = 0; u < NL; ++u) v[u] = __ldcg(src + (long long)u * stride + threadIdx.x);
  double s = 0;
#pragma unroll
  for (int u = 0; u < NL; ++u) s += v[u];
  __syncthreads();
  long long t1 = clock64();
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double *out, *src;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&src, 64 << 20);
  cudaMemset(src, 0, 64 << 20);
  cudaMallocManaged(&cyc, 1024 * sizeof(long long));
  const int iters = 1000;
  for (int rep = 0; rep < 2; ++rep) {
    k_chain<1><<<1, 32>>>(out, cyc, iters); cudaDeviceSynchronize();
    printf("DMMA 1 warp, 1 chain: %.1f cycles/dmma (latency)\n", (double)cyc[0] / iters);
    k_chain<4><<<1, 32>>>(out, cyc, iters); cudaDeviceSynchronize();
    printf("DMMA 1 warp, 4 chains: %.1f cycles/dmma\n", (double)cyc[0] / iters / 4);
    k_chain<1><<<1, 256>>>(out, cyc, iters); cudaDeviceSynchronize();
    printf("DMMA 8 warps, 1 chain each: %.1f cycles per dmma-round (8 dmma)\n", (double)cyc[0] / iters);
    k_chain<4><<<1, 256>>>(out, cyc, iters); cudaDeviceSynchronize();
    printf("DMMA 8 warps, 4 chains each: %.1f cycles per 32 dmma -> %.2f cycles/dmma/SM\n", (double)cyc[0] / iters, (double)cyc[0] / iters / 32);
    k_ffma<<<1, 256>>>(out, cyc, iters); cudaDeviceSynchronize();
    printf("DFMA 8 warps x 8 chains: %.2f cycles per warp-instr/SM\n", (double)cyc[0] / iters / 64);
    // L2-resident loads (warm them first)
    k_loads<80><<<1, 256>>>(src, out, cyc, 4096); cudaDeviceSynchronize();
    k_loads<80><<<1, 256>>>(src, out, cyc, 4096); cudaDeviceSynchronize();
    printf("80 ld.cg per thread (256 thr, L2-resident): %lld cycles\n", cyc[0]);
    k_loads<8><<<1, 256>>>(src, out, cyc, 4096); cudaDeviceSynchronize();
    printf("8 ld.cg per thread: %lld cycles\n", cyc[0]);
    k_loads<1><<<1, 256>>>(src, out, cyc, 4096); cudaDeviceSynchronize();
    printf("1 ld.cg per thread: %lld cycles\n", cyc[0]);
  }
  return 0;
}
