// Microbenchmark: cluster barrier latency, DSMEM remote-read latency/bandwidth vs the global
// (atomic + spin) team barrier. nvcc -O3 -gencode arch=compute_100a,code=sm_100a cluster_bench.cu
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__global__ void k_cbar(long long* cyc, int iters) {
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) cyc[0] = (t1 - t0) / iters;
}
__global__ void k_dsmem(long long* cyc, double* out, int iters, int nread) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i * 1e-3 + cl.block_rank();
  cl.sync();
  const unsigned peer = (cl.block_rank() + 1) % cl.num_blocks();
  double* rem = cl.map_shared_rank(sm, peer);
  double s = 0.0;
  // dependent chain latency
  long long t0 = clock64();
  int idx = threadIdx.x & 7;
  for (int i = 0; i < iters; ++i) {
    const double v = rem[idx];
    s += v;
    idx = ((int)v + i) & 7;
  }
  long long t1 = clock64();
  // bandwidth: every thread reads nread doubles
  __syncthreads();
  long long t2 = clock64();
  for (int r = 0; r < nread; ++r) s += rem[(threadIdx.x + r * blockDim.x) & 8191];
  __syncthreads();
  long long t3 = clock64();
  cl.sync();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && cl.block_rank() == 0) {
    cyc[1] = (t1 - t0) / iters;
    cyc[2] = t3 - t2;
  }
}
struct Hdr { unsigned count, gen; };
__global__ void k_gbar(Hdr* h, long long* cyc, int iters, int P) {
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
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
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[3] = (t1 - t0) / iters;
}
int main() {
  long long* cyc;
  double* out;
  Hdr* h;
  cudaMallocManaged(&cyc, 8 * sizeof(long long));
  cudaMalloc(&out, 1 << 24);
  cudaMalloc(&h, sizeof(Hdr));
  for (int C : {2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(256);
    if (C > 8) {
      cudaFuncSetAttribute(k_cbar, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    }
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_cbar, cyc, 1000);
    cudaDeviceSynchronize();
    if (e) printf("C=%d cbar launch: %s\n", C, cudaGetErrorString(e));
    cfg.dynamicSmemBytes = 8192 * sizeof(double);
    cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 * 8);
    e = cudaLaunchKernelEx(&cfg, k_dsmem, cyc, out, 1000, 64);
    cudaError_t e2 = cudaDeviceSynchronize();
    if (e || e2) printf("C=%d dsmem: %s %s\n", C, cudaGetErrorString(e), cudaGetErrorString(e2));
    cudaMemset(h, 0, sizeof(Hdr));
    void* args[] = {&h, &cyc, nullptr, nullptr};
    int iters = 1000;
    args[2] = &iters;
    args[3] = &C;
    cudaLaunchCooperativeKernel((void*)k_gbar, dim3(C), dim3(256), args, 0, 0);
    cudaDeviceSynchronize();
    printf("C=%2d: cluster.sync %lld cycles | DSMEM dependent read %lld cycles | 64 reads x 256 thr (128 KB) %lld cycles | global team barrier %lld cycles\n",
           C, cyc[0], cyc[1], cyc[2], cyc[3]);
  }
  int maxc = 0;
  {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 16; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1; cfg.gridDim = dim3(16 * 20); cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 200 * 1024;
    cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaOccupancyMaxActiveClusters(&maxc, (void*)k_dsmem, &cfg);
    printf("max active clusters of 16 with 200 KB smem: %d\n", maxc);
    at[0].val.clusterDim.x = 8; cfg.gridDim = dim3(8 * 20);
    cudaOccupancyMaxActiveClusters(&maxc, (void*)k_dsmem, &cfg);
    printf("max active clusters of 8 with 200 KB smem: %d\n", maxc);
  }
  return 0;
}
