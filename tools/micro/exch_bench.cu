// Row-exchange microbenchmark on a thread-block cluster: every CTA owns n values per step and
// must deliver them to every CTA of the cluster (all-gather of C*n doubles per step), double
// buffered, completion on the receiver's mbarrier.
//  mode 0: one st.async (8 bytes) per value and destination (the k_gid_cpqr scheme)
//  mode 1: values staged in local shared memory, one cp.async.bulk per destination
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o exch_bench exch_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, unsigned rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const uint32_t a = smem_addr(bar);
  unsigned ok = 0;
  while (!ok)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(a), "r"(parity) : "memory");
}
template <int MODE>
__global__ void __launch_bounds__(256, 1) k(int C, int n, int steps, long long* cyc, double* out) {
  __shared__ __align__(16) double rowbuf[2][1024];
  __shared__ __align__(16) double stage[2][64];
  __shared__ __align__(8) uint64_t mbar[2];
  const int tid = threadIdx.x, c = (int)cluster_rank();
  const int np = (n + 1) & ~1;   // padded segment
  if (tid == 0) {
    for (int q = 0; q < 2; ++q)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(mbar + q)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cluster_barrier();
  const uint32_t rb = smem_addr(&rowbuf[0][0]), bar = smem_addr(mbar);
  double acc = 0.0;
  long long t0 = clock64(), tp = 0, tw = 0;
  for (int i = 0; i < steps; ++i) {
    const int q = i & 1;
    long long a0 = clock64();
    if (tid == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar + 8u * q), "r"(8u * (unsigned)(C * np)) : "memory");
    if (MODE == 0) {
      // tpc threads per value, each pushing to C / tpc destinations
      const int tpc = 8;
      const int part = tid % tpc;
      for (int lb = tid / tpc; lb < np; lb += 256 / tpc) {
        const double v = acc + lb + i;
        for (int u = 0; u * tpc + part < C; ++u) {
          const unsigned dst = u * tpc + part;
          const uint32_t ra = mapa_u32(rb, dst) + (uint32_t)(q * 1024 + c * np + lb) * 8u;
          const uint32_t rbar = mapa_u32(bar, dst) + 8u * q;
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(ra),
                       "l"(__double_as_longlong(v)), "r"(rbar) : "memory");
        }
      }
    } else {
      if (tid < np) stage[q][tid] = acc + tid + i;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid < C) {
        const uint32_t ra = mapa_u32(rb, tid) + (uint32_t)(q * 1024 + c * np) * 8u;
        const uint32_t rbar = mapa_u32(bar, tid) + 8u * q;
        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(ra),
                     "r"(smem_addr(&stage[q][0])), "r"(8u * (unsigned)np), "r"(rbar) : "memory");
      }
    }
    long long a1 = clock64();
    mbar_wait(mbar + q, (unsigned)((i >> 1) & 1));
    long long a2 = clock64();
    tp += a1 - a0;
    tw += a2 - a1;
    // consume: every thread reads a few entries (dependency for the next step)
    acc = rowbuf[q][(tid * 3) % (C * np)] * 1e-9;
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0 && c == 0 && blockIdx.x < C) {
    cyc[0] = (t1 - t0) / steps;
    cyc[1] = tp / steps;
    cyc[2] = tw / steps;
  }
  out[blockIdx.x * 256 + tid] = acc;
  cluster_barrier();
}
template <int MODE>
void run(int C, int n, int ncl) {
  long long* cyc;
  double* out;
  cudaMallocManaged(&cyc, 64);
  cudaMalloc(&out, 8 * 256 * 256);
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cfg.gridDim = dim3(C * ncl); cfg.blockDim = dim3(256);
  for (int rep = 0; rep < 2; ++rep) {
    cudaError_t e = cudaLaunchKernelEx(&cfg, k<MODE>, C, n, 2000, cyc, out);
    if (e != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) { printf("error %s\n", cudaGetErrorString(cudaGetLastError())); return; }
  }
  printf("mode %d C %2d n %2d clusters %d: %lld cycles/step (push %lld wait %lld)\n", MODE, C, n, ncl, cyc[0], cyc[1], cyc[2]);
  fflush(stdout);
  cudaFree(cyc); cudaFree(out);
}
int main() {
  for (int ncl : {1, 8})
    for (int C : {4, 16})
      for (int n : {13, 31, 56}) {
        if (C * ((n + 1) & ~1) > 1024) continue;
        run<0>(C, n, ncl);
        run<1>(C, n, ncl);
      }
  return 0;
}
