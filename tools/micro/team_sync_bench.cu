// Microbenchmark: latency of a per-team software barrier among co-resident CTAs.
#include <cstdio>
#include <cuda_runtime.h>
struct Hdr { unsigned count, gen; double pad; };

__device__ void sync_volatile(Hdr* h, int P) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vg = &h->gen;
    unsigned g0 = *vg;
    __threadfence();
    if (atomicAdd(&h->count, 1u) == (unsigned)(P - 1)) { h->count = 0; __threadfence(); atomicAdd(&h->gen, 1u); }
    else while (*vg == g0) __nanosleep(40);
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) {
  unsigned old; asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory"); return old;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
// generation barrier: arrivals counted on `count`, the last arriver bumps `gen`
__device__ void sync_acqrel(Hdr* h, int P, unsigned& gen_local) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned target = gen_local + 1;
    if (atom_add_acqrel(&h->count, 1u) == (unsigned)(P - 1)) {
      h->count = 0;
      st_release(&h->gen, target);
    } else {
      while (ld_acquire(&h->gen) != target) {}
    }
    gen_local = target;
  }
  __syncthreads();
}

__global__ void bench(Hdr* hdr, int P, int iters, int mode, long long* out) {
  const int team = blockIdx.x / P;
  Hdr* h = hdr + team;
  unsigned gl = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (mode == 0) sync_volatile(h, P); else sync_acqrel(h, P, gl);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int mode = 0; mode < 2; ++mode)
    for (int P : {2, 8, 29, 64}) {
      int teams = 145 / P; if (teams < 1) teams = 1;
      Hdr* h; cudaMalloc(&h, teams * sizeof(Hdr)); cudaMemset(h, 0, teams * sizeof(Hdr));
      long long* o; cudaMalloc(&o, teams * P * sizeof(long long));
      const int iters = 2000;
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      void* args[] = {&h, &P, (void*)&iters, &mode, &o};
      int it = iters;
      args[2] = &it;
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)bench, dim3(teams * P), dim3(256), args, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("mode %s P=%3d teams=%2d: %.2f us per barrier (err=%s)\n", mode ? "acq_rel " : "volatile", P, teams,
             1e3 * ms / iters, cudaGetErrorString(cudaGetLastError()));
      cudaFree(h); cudaFree(o);
    }
  return 0;
}
