// Device-side level-0 planner.
//
// Computes on the GPU, from the spec and the device CSR pattern of A, exactly what the host
// planner (planner.cpp: classify_all + pattern_from_csr + build_level) computes for level 0:
//
//   * groups in classify order (hierarchy.py:124-133: key = x-major cell index, kind bits last;
//     members ascending, hierarchy.py:145): one stable radix sort of the DOFs by key;
//   * the symbolic block pattern: stencil group pairs (one per nnz, sorted + unique) plus the
//     elimination fill (every pair of boundary groups of a cell), blocks numbered in
//     (g, h) order, the symmetric adjacency sorted by neighbour, pool offsets;
//   * cell boundary lists, the Schur-target contribution lists (per target block, its cells in
//     cell order = the fixed summation order of k_schur), the block-Jacobi scaling blocks;
//   * skeleton neighbour lists and the dependency counts / successor lists of the sequential
//     skeletonization.
//
// The arrays stay on the device for the level-0 kernels (DevPlan0); only what the host level
// loop reads afterwards is copied back (group lists, block pairs, cell lists, scaling blocks,
// skeleton neighbour lists). The dependency wavefronts (a sequential longest-path pass) are
// computed on the host from the downloaded neighbour lists. tests/test_gpu_planner.py checks
// every array against the host planner (phif_plan_check).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <mutex>
#include <tuple>
#include <cstring>

#include "engine.h"
#include "gpu_plan.h"

namespace phif {

extern std::atomic<long long> g_launches;

namespace {

#define GCK(x)                                                                                   \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess) throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));    \
  } while (0)

constexpr unsigned long long SENT = ~0ull;
constexpr int TPB = 256;

inline int nblk(int64_t n) { return (int)std::max<int64_t>(1, (n + TPB - 1) / TPB); }
inline int bits_for(int64_t v) {   // bits needed to represent values in [0, v]
  int b = 1;
  while (b < 63 && (int64_t(1) << b) <= v) ++b;
  return b;
}

template <class T>
T* A_(DBuf& b) {
  return b.as<T>();
}

template <class T>
void alloc_n(DBuf& b, int64_t n, cudaStream_t s) {
  b.alloc((size_t)std::max<int64_t>(n, 1) * sizeof(T), s);
}

template <class T>
T read1(const T* d, cudaStream_t s) {
  T h;
  GCK(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, s));
  GCK(cudaStreamSynchronize(s));
  return h;
}

inline void pool_take(std::vector<int>& h, int64_t n) { h = pool_take_int((size_t)n); }
inline void pool_take(std::vector<int64_t>& h, int64_t n) { h = pool_take_i64((size_t)n); }

template <class T>
void down(std::vector<T>& h, const DBuf& d, int64_t n, cudaStream_t s) {
  pool_take(h, n);   // recycled host allocation (no page faults once warm)
  if (n) download_bytes(h.data(), d.p, (size_t)n * sizeof(T), s);
}

// ---------------------------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------------------------
__global__ void k_p0_keys(int dim, int n, int m, int64_t N, int* keys, int* vals) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const int64_t side = n - 1;
  int c[3];
  c[0] = (int)(i % side) + 1;
  c[1] = (int)((i / side) % side) + 1;
  c[2] = dim == 3 ? (int)(i / (side * side)) + 1 : 0;
  const int per = n / m;
  int64_t key = 0;
  int bits = 0;
  for (int d = 0; d < dim; ++d) {
    key = key * per + c[d] / m;
    if (c[d] % m == 0) bits |= 1 << d;
  }
  keys[i] = (int)((key << dim) | bits);
  vals[i] = (int)i;
}

__global__ void k_p0_heads(const int* skeys, int64_t N, int* head) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= N) return;
  head[p] = (p == 0 || skeys[p] != skeys[p - 1]) ? 1 : 0;
}

__global__ void k_p0_groups(const int* skeys, const int* seg, const int* head, const int* mem, int64_t N, int dim,
                            int64_t* goff, int* gkey, int* gid) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= N) return;
  const int g = seg[p] - 1;
  if (head[p]) {
    goff[g] = p;
    gkey[g] = skeys[p];
  }
  if (p == N - 1) goff[g + 1] = N;
  gid[mem[p]] = g;
  (void)dim;
}

__global__ void k_p0_gattr(const int64_t* goff, const int* gkey, int G, int dim, int* gsize, int* kind, uint8_t* fint,
                           uint8_t* fnint, uint8_t* fsep) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= G) return;
  gsize[g] = (int)(goff[g + 1] - goff[g]);
  const int kd = __popc(gkey[g] & ((1 << dim) - 1));
  kind[g] = kd;
  fint[g] = kd == 0;
  fnint[g] = kd != 0;
  fsep[g] = kd == 1;
}

// one candidate pair per nnz (row group <= column group), plus (g, g) for every group
__global__ void k_p0_stencil_pairs(const int64_t* rowptr, const int* col, const int* gid, int64_t N, int G,
                                   unsigned long long* out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < N) {
    const unsigned long long gr = (unsigned)gid[r];
    for (int64_t e = rowptr[r]; e < rowptr[r + 1]; ++e) {
      const unsigned long long gc = (unsigned)gid[col[e]];
      out[e] = gr <= gc ? ((gr << 32) | gc) : SENT;
    }
  }
  if (r < G) out[rowptr[N] + r] = ((unsigned long long)r << 32) | (unsigned long long)r;
}

// row starts of a sorted (first << 32 | second) list: off[first] = first index (every row present)
__global__ void k_p0_row_starts(const unsigned long long* keys, int64_t n, int G, int64_t* off) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const int f = (int)(keys[q] >> 32);
  if (q == 0 || (int)(keys[q - 1] >> 32) != f) off[f] = q;
  if (q == n - 1) off[G] = n;
}

__global__ void k_p0_sk_index(const int* skeleton, int nsk, int* sk_index) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nsk) sk_index[skeleton[i]] = i;
}

// cells: neighbour counts (stencil upper list minus the interior itself) + closure checks
__global__ void k_p0_cell_counts(const int* interior, int p, const int64_t* ust_off, const unsigned long long* ust,
                                 const int* kind, int64_t* ncnt, int64_t* pcnt, int* bad) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= p) return;
  const int I = interior[t];
  const int64_t a = ust_off[I], e = ust_off[I + 1];
  if ((int)(ust[a] & 0xffffffffu) != I) atomicMax(bad, 1);   // interior not first in its closure
  for (int64_t q = a + 1; q < e; ++q)
    if (kind[(int)(ust[q] & 0xffffffffu)] == 0) atomicMax(bad, 2);   // two interior groups coupled
  const int64_t nt = e - a - 1;
  ncnt[t] = nt;
  pcnt[t] = nt * (nt + 1) / 2;
}

// cell lists + fill-pair emission (all pairs a <= b of the cell's boundary groups)
__global__ void k_p0_cell_fill(const int* interior, int p, const int64_t* ust_off, const unsigned long long* ust,
                               const int64_t* noff, const int64_t* poff, const int* gsize, int* cell_nbr,
                               int* cell_nbr_col, int* cell_nbr_w, int* cell_n, int* cell_b, unsigned long long* fill) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= p) return;
  const int I = interior[t];
  const int64_t a = ust_off[I] + 1, e = ust_off[I + 1];
  const int64_t o = noff[t];
  int bc = 0;
  for (int64_t q = a; q < e; ++q) {
    const int h = (int)(ust[q] & 0xffffffffu);
    cell_nbr[o + (q - a)] = h;
    cell_nbr_col[o + (q - a)] = bc;
    cell_nbr_w[o + (q - a)] = gsize[h];
    bc += gsize[h];
  }
  cell_n[t] = gsize[I];
  cell_b[t] = bc;
  int64_t f = poff[t];
  for (int64_t i = a; i < e; ++i) {
    const unsigned long long gi = ust[i] & 0xffffffffu;
    for (int64_t j = i; j < e; ++j) fill[f++] = (gi << 32) | (ust[j] & 0xffffffffu);
  }
}

__global__ void k_p0_blocks(const unsigned long long* keys, int64_t nb, const int* gsize, int* bg, int* bh,
                            int64_t* bsz, unsigned long long* adj_keys, int* adj_val, uint8_t* fscale,
                            const int* kind) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nb) return;
  const int g = (int)(keys[q] >> 32), h = (int)(keys[q] & 0xffffffffu);
  bg[q] = g;
  bh[q] = h;
  bsz[q] = (int64_t)gsize[g] * gsize[h];
  adj_keys[2 * q] = keys[q];
  adj_val[2 * q] = (int)q;
  adj_keys[2 * q + 1] = g != h ? (((unsigned long long)h << 32) | (unsigned long long)g) : SENT;
  adj_val[2 * q + 1] = (int)q;
  fscale[q] = g != h && kind[g] != 0 && kind[h] != 0;
}

__global__ void k_p0_adj(const unsigned long long* skeys, int64_t nadj, int G, int* adj_nbr, int64_t* adj_off) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nadj) return;
  const int r = (int)(skeys[k] >> 32);
  adj_nbr[k] = (int)(skeys[k] & 0xffffffffu);
  if (k == 0 || (int)(skeys[k - 1] >> 32) != r) adj_off[r] = k;
  if (k == nadj - 1) adj_off[G] = nadj;
}

__global__ void k_p0_diag(const int64_t* uoff, int G, int* diag) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g < G) diag[g] = (int)uoff[g];
}

__global__ void k_p0_cell_blk(const int* interior, int p, const int64_t* uoff, const int64_t* noff,
                              const int64_t* ust_off, int* cell_nbr_blk, int* bad) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= p) return;
  const int I = interior[t];
  const int64_t nt = noff[t + 1] - noff[t];
  if (uoff[I + 1] - uoff[I] != ust_off[I + 1] - ust_off[I]) atomicMax(bad, 3);   // (fill of an interior row)
  for (int64_t j = 0; j < nt; ++j) cell_nbr_blk[noff[t] + j] = (int)(uoff[I] + 1 + j);
}

// Schur contributions: for every cell t and boundary pair (a_i, a_j), i <= j: key (block, t)
__global__ void k_p0_schur_emit(int p, const int64_t* noff, const int64_t* poff, const int* cell_nbr,
                                const int* cell_nbr_col, const int64_t* uoff, const int* bh,
                                unsigned long long* keys, int* crow, int* ccol, int* idx) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= p) return;
  const int64_t a = noff[t], e = noff[t + 1];
  int64_t f = poff[t];
  for (int64_t i = a; i < e; ++i) {
    const int gi = cell_nbr[i];
    const int* lo = bh + uoff[gi];
    const int* hi = bh + uoff[gi + 1];
    for (int64_t j = i; j < e; ++j) {
      const int gj = cell_nbr[j];
      // lower bound of gj in the (ascending) upper list of gi
      const int* l = lo;
      int64_t len = hi - lo;
      while (len > 0) {
        const int64_t half = len >> 1;
        if (l[half] < gj) {
          l += half + 1;
          len -= half + 1;
        } else {
          len = half;
        }
      }
      const int64_t blk = uoff[gi] + (l - lo);
      keys[f] = ((unsigned long long)blk << 32) | (unsigned long long)t;
      crow[f] = cell_nbr_col[i];
      ccol[f] = cell_nbr_col[j];
      idx[f] = (int)f;
      ++f;
    }
  }
}

__global__ void k_p0_schur_out(const unsigned long long* skeys, const int* sidx, const int* crow, const int* ccol,
                               int64_t ne, int* con_cell, int* con_row, int* con_col, int* head) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= ne) return;
  con_cell[k] = (int)(skeys[k] & 0xffffffffu);
  con_row[k] = crow[sidx[k]];
  con_col[k] = ccol[sidx[k]];
  head[k] = (k == 0 || (skeys[k] >> 32) != (skeys[k - 1] >> 32)) ? 1 : 0;
}

__global__ void k_p0_tgt(const unsigned long long* skeys, const int* seg, const int* head, int64_t ne, int* tgt_blk,
                         int64_t* tgt_off) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= ne) return;
  if (head[k]) {
    const int j = seg[k] - 1;
    tgt_blk[j] = (int)(skeys[k] >> 32);
    tgt_off[j] = k;
  }
  if (k == ne - 1) tgt_off[seg[k]] = ne;
}

__global__ void k_p0_sk_counts(const int* skeleton, int nsk, const int64_t* adj_off, const int* adj_nbr,
                               const int* kind, const int* sk_index, int64_t* ncnt, int* ndep, int64_t* scnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nsk) return;
  const int gg = skeleton[i];
  int64_t c = 0, sc = 0;
  int nd = 0;
  for (int64_t q = adj_off[gg]; q < adj_off[gg + 1]; ++q) {
    const int h = adj_nbr[q];
    if (h == gg || kind[h] == 0) continue;
    ++c;
    const int j = sk_index[h];
    if (j >= 0 && j < i) ++nd;
    if (j > i) ++sc;
  }
  ncnt[i] = c;
  ndep[i] = nd;
  scnt[i] = sc;
}

__global__ void k_p0_sk_fill(const int* skeleton, int nsk, const int64_t* adj_off, const int* adj_nbr,
                             const int* adj_blk, const int* kind, const int* sk_index, const int64_t* noff,
                             const int64_t* soff, int* sk_nbr, int* sk_nbr_blk, int* sk_succ) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nsk) return;
  const int gg = skeleton[i];
  int64_t o = noff[i], so = soff[i];
  for (int64_t q = adj_off[gg]; q < adj_off[gg + 1]; ++q) {
    const int h = adj_nbr[q];
    if (h == gg || kind[h] == 0) continue;
    sk_nbr[o] = h;
    sk_nbr_blk[o++] = adj_blk[q];
    if (sk_index[h] > i) sk_succ[so++] = sk_index[h];
  }
}

// ---------------------------------------------------------------------------------------------
// host helpers (CUB two-phase calls with cached temporary storage)
// ---------------------------------------------------------------------------------------------
struct Temp {
  DBuf buf;
  cudaStream_t s;
  void* get(size_t bytes) {
    if (bytes > buf.bytes) buf.alloc(bytes, s);
    return buf.p;
  }
};

void scan_incl(const int* in, int* out, int64_t n, Temp& tmp, cudaStream_t s) {
  size_t b = 0;
  GCK(cub::DeviceScan::InclusiveSum(nullptr, b, in, out, n, s));
  GCK(cub::DeviceScan::InclusiveSum(tmp.get(b), b, in, out, n, s));
}

// exclusive prefix of n counts into off[0..n] (off[n] = total, returned)
int64_t offsets(const DBuf& cnt, DBuf& off, int64_t n, Temp& tmp, cudaStream_t s) {
  alloc_n<int64_t>(off, n + 1, s);
  GCK(cudaMemsetAsync(off.p, 0, sizeof(int64_t), s));
  if (n == 0) return 0;
  size_t b = 0;
  GCK(cub::DeviceScan::InclusiveSum(nullptr, b, cnt.as<int64_t>(), off.as<int64_t>() + 1, n, s));
  GCK(cub::DeviceScan::InclusiveSum(tmp.get(b), b, cnt.as<int64_t>(), off.as<int64_t>() + 1, n, s));
  return read1(off.as<int64_t>() + n, s);
}

// indices g in [0, n) with flag[g] != 0, in order
int select_idx(const uint8_t* flags, int n, DBuf& out, Temp& tmp, DBuf& cnt, cudaStream_t s) {
  alloc_n<int>(out, n, s);
  size_t b = 0;
  thrust::counting_iterator<int> it(0);
  GCK(cub::DeviceSelect::Flagged(nullptr, b, it, flags, out.as<int>(), cnt.as<int>(), n, s));
  GCK(cub::DeviceSelect::Flagged(tmp.get(b), b, it, flags, out.as<int>(), cnt.as<int>(), n, s));
  return read1(cnt.as<int>(), s);
}

// sort 64-bit keys (bits [0, end_bit)) and keep the distinct ones (sentinels dropped); returns count
int64_t sort_unique(DBuf& keys, int64_t n, int end_bit, DBuf& out, Temp& tmp, DBuf& cnt, cudaStream_t s) {
  DBuf sorted;
  alloc_n<unsigned long long>(sorted, n, s);
  size_t b = 0;
  const auto* k = keys.as<unsigned long long>();
  auto* ks = sorted.as<unsigned long long>();
  GCK(cub::DeviceRadixSort::SortKeys(nullptr, b, k, ks, n, 0, 64, s));
  GCK(cub::DeviceRadixSort::SortKeys(tmp.get(b), b, k, ks, n, 0, 64, s));
  (void)end_bit;
  alloc_n<unsigned long long>(out, n, s);
  b = 0;
  GCK(cub::DeviceSelect::Unique(nullptr, b, ks, out.as<unsigned long long>(), cnt.as<int>(), n, s));
  GCK(cub::DeviceSelect::Unique(tmp.get(b), b, ks, out.as<unsigned long long>(), cnt.as<int>(), n, s));
  int64_t m = read1(cnt.as<int>(), s);
  if (m > 0 && read1(out.as<unsigned long long>() + m - 1, s) == SENT) --m;
  return m;
}

}  // namespace

bool gpu_plan0_applicable(const Spec& s, int big_cell) {
  int64_t n = 1;
  for (int d = 0; d < s.dim; ++d) n *= (s.m - 1);
  if (n < big_cell) return true;   // level-0 cells on the one-CTA path
  // 2D cells on the banded (or tile-parallel) path: their host work lists come from the downloaded plan
  // (PHIF_HOST_PLAN_2D=1 keeps the host planner for them)
  static const bool host2d = getenv("PHIF_HOST_PLAN_2D") != nullptr;
  return !host2d && s.dim == 2;
}

void plan_level0_device(const Spec& s, const int64_t* rowptr, const int* col, int64_t nnz, LevelPlan& lp,
                        DevPlan0& dp, cudaStream_t st) {
  static const bool tdbg = getenv("PHIF_PLAN_TIMING") != nullptr;
  auto tl = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!tdbg) return;
    cudaStreamSynchronize(st);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "  [gpu plan L0] %-28s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(now - tl).count());
    tl = now;
  };
  Temp tmp{DBuf(), st};
  DBuf cnt;
  alloc_n<int>(cnt, 2, st);
  const int64_t N = s.N;
  const int dim = s.dim;
  int nlaunch = 0;
  auto L = [&]() { ++nlaunch; };
  // ---- groups --------------------------------------------------------------------------------
  const int per = s.n / s.m;
  int64_t nkeys = 1;
  for (int d = 0; d < dim; ++d) nkeys *= per;
  nkeys <<= dim;
  DBuf keys, vals, skeys, head, seg, gid, gkey;
  alloc_n<int>(keys, N, st);
  alloc_n<int>(vals, N, st);
  alloc_n<int>(skeys, N, st);
  alloc_n<int>(dp.mem, N, st);
  alloc_n<int>(head, N, st);
  alloc_n<int>(seg, N, st);
  alloc_n<int>(gid, N, st);
  k_p0_keys<<<nblk(N), TPB, 0, st>>>(dim, s.n, s.m, N, keys.as<int>(), vals.as<int>());
  L();
  {
    size_t b = 0;
    const int eb = bits_for(nkeys - 1);
    GCK(cub::DeviceRadixSort::SortPairs(nullptr, b, keys.as<int>(), skeys.as<int>(), vals.as<int>(),
                                        dp.mem.as<int>(), N, 0, eb, st));
    GCK(cub::DeviceRadixSort::SortPairs(tmp.get(b), b, keys.as<int>(), skeys.as<int>(), vals.as<int>(),
                                        dp.mem.as<int>(), N, 0, eb, st));
  }
  k_p0_heads<<<nblk(N), TPB, 0, st>>>(skeys.as<int>(), N, head.as<int>());
  L();
  scan_incl(head.as<int>(), seg.as<int>(), N, tmp, st);
  const int G = read1(seg.as<int>() + N - 1, st);
  alloc_n<int64_t>(dp.goff, G + 1, st);
  alloc_n<int>(gkey, G, st);
  k_p0_groups<<<nblk(N), TPB, 0, st>>>(skeys.as<int>(), seg.as<int>(), head.as<int>(), dp.mem.as<int>(), N, dim,
                                        dp.goff.as<int64_t>(), gkey.as<int>(), gid.as<int>());
  L();
  DBuf fint, fnint, fsep;
  alloc_n<int>(dp.gsize, G, st);
  alloc_n<int>(dp.kind, G, st);
  alloc_n<uint8_t>(fint, G, st);
  alloc_n<uint8_t>(fnint, G, st);
  alloc_n<uint8_t>(fsep, G, st);
  k_p0_gattr<<<nblk(G), TPB, 0, st>>>(dp.goff.as<int64_t>(), gkey.as<int>(), G, dim, dp.gsize.as<int>(),
                                       dp.kind.as<int>(), fint.as<uint8_t>(), fnint.as<uint8_t>(), fsep.as<uint8_t>());
  L();
  const int p = select_idx(fint.as<uint8_t>(), G, dp.interior, tmp, cnt, st);
  const int r = select_idx(fnint.as<uint8_t>(), G, dp.precond, tmp, cnt, st);
  const int nsk = select_idx(fsep.as<uint8_t>(), G, dp.skeleton, tmp, cnt, st);
  lap("groups");
  // ---- stencil pattern -----------------------------------------------------------------------
  DBuf cand, ust, ust_off;
  alloc_n<unsigned long long>(cand, nnz + G, st);
  k_p0_stencil_pairs<<<nblk(std::max<int64_t>(N, G)), TPB, 0, st>>>(rowptr, col, gid.as<int>(), N, G,
                                                                      cand.as<unsigned long long>());
  L();
  const int64_t nst = sort_unique(cand, nnz + G, 64, ust, tmp, cnt, st);
  cand.release();
  lap("stencil pairs");
  alloc_n<int64_t>(ust_off, G + 1, st);
  k_p0_row_starts<<<nblk(nst), TPB, 0, st>>>(ust.as<unsigned long long>(), nst, G, ust_off.as<int64_t>());
  L();
  // ---- cells + fill --------------------------------------------------------------------------
  DBuf ncnt, pcnt, poff, bad;
  alloc_n<int64_t>(ncnt, p, st);
  alloc_n<int64_t>(pcnt, p, st);
  alloc_n<int>(bad, 1, st);
  GCK(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
  k_p0_cell_counts<<<nblk(p), TPB, 0, st>>>(dp.interior.as<int>(), p, ust_off.as<int64_t>(),
                                             ust.as<unsigned long long>(), dp.kind.as<int>(), ncnt.as<int64_t>(),
                                             pcnt.as<int64_t>(), bad.as<int>());
  L();
  const int64_t ncn = offsets(ncnt, dp.cell_nbr_off, p, tmp, st);
  const int64_t nfill = offsets(pcnt, poff, p, tmp, st);
  alloc_n<int>(dp.cell_nbr, ncn, st);
  alloc_n<int>(dp.cell_nbr_col, ncn, st);
  alloc_n<int>(dp.cell_nbr_w, ncn, st);
  alloc_n<int>(dp.cell_nbr_blk, ncn, st);
  alloc_n<int>(dp.cell_n, p, st);
  alloc_n<int>(dp.cell_b, p, st);
  DBuf fillk, blocks;
  alloc_n<unsigned long long>(fillk, nfill + nst, st);
  k_p0_cell_fill<<<nblk(p), TPB, 0, st>>>(dp.interior.as<int>(), p, ust_off.as<int64_t>(),
                                           ust.as<unsigned long long>(), dp.cell_nbr_off.as<int64_t>(),
                                           poff.as<int64_t>(), dp.gsize.as<int>(), dp.cell_nbr.as<int>(),
                                           dp.cell_nbr_col.as<int>(), dp.cell_nbr_w.as<int>(), dp.cell_n.as<int>(),
                                           dp.cell_b.as<int>(), fillk.as<unsigned long long>());
  L();
  GCK(cudaMemcpyAsync(fillk.as<unsigned long long>() + nfill, ust.p, nst * sizeof(unsigned long long),
                      cudaMemcpyDeviceToDevice, st));
  const int64_t nb = sort_unique(fillk, nfill + nst, 64, blocks, tmp, cnt, st);
  fillk.release();
  lap("fill pairs");
  // ---- blocks, adjacency, pool ---------------------------------------------------------------
  DBuf uoff, bsz, adjk, adjv, adjks, fscale;
  alloc_n<int64_t>(uoff, G + 1, st);
  k_p0_row_starts<<<nblk(nb), TPB, 0, st>>>(blocks.as<unsigned long long>(), nb, G, uoff.as<int64_t>());
  L();
  alloc_n<int>(dp.bg, nb, st);
  alloc_n<int>(dp.bh, nb, st);
  alloc_n<int64_t>(bsz, nb, st);
  alloc_n<unsigned long long>(adjk, 2 * nb, st);
  alloc_n<int>(adjv, 2 * nb, st);
  alloc_n<uint8_t>(fscale, nb, st);
  k_p0_blocks<<<nblk(nb), TPB, 0, st>>>(blocks.as<unsigned long long>(), nb, dp.gsize.as<int>(), dp.bg.as<int>(),
                                         dp.bh.as<int>(), bsz.as<int64_t>(), adjk.as<unsigned long long>(),
                                         adjv.as<int>(), fscale.as<uint8_t>(), dp.kind.as<int>());
  L();
  const int64_t nadj = 2 * nb - G;
  alloc_n<unsigned long long>(adjks, 2 * nb, st);
  alloc_n<int>(dp.adj_blk, 2 * nb, st);
  {
    size_t b = 0;
    GCK(cub::DeviceRadixSort::SortPairs(nullptr, b, adjk.as<unsigned long long>(), adjks.as<unsigned long long>(),
                                        adjv.as<int>(), dp.adj_blk.as<int>(), 2 * nb, 0, 64, st));
    GCK(cub::DeviceRadixSort::SortPairs(tmp.get(b), b, adjk.as<unsigned long long>(), adjks.as<unsigned long long>(),
                                        adjv.as<int>(), dp.adj_blk.as<int>(), 2 * nb, 0, 64, st));
  }
  alloc_n<int>(dp.adj_nbr, nadj, st);
  alloc_n<int64_t>(dp.adj_off, G + 1, st);
  k_p0_adj<<<nblk(nadj), TPB, 0, st>>>(adjks.as<unsigned long long>(), nadj, G, dp.adj_nbr.as<int>(),
                                        dp.adj_off.as<int64_t>());
  L();
  adjk.release();
  adjv.release();
  adjks.release();
  alloc_n<int>(dp.diag_blk, G, st);
  k_p0_diag<<<nblk(G), TPB, 0, st>>>(uoff.as<int64_t>(), G, dp.diag_blk.as<int>());
  L();
  lp.pool_doubles = offsets(bsz, dp.boff, nb, tmp, st);
  lap("adjacency + pool");
  k_p0_cell_blk<<<nblk(p), TPB, 0, st>>>(dp.interior.as<int>(), p, uoff.as<int64_t>(), dp.cell_nbr_off.as<int64_t>(),
                                          ust_off.as<int64_t>(), dp.cell_nbr_blk.as<int>(), bad.as<int>());
  L();
  // ---- Schur targets -------------------------------------------------------------------------
  {
    DBuf sk, crow, ccol, sidx, sks, sidx2, hd, sg;
    alloc_n<unsigned long long>(sk, nfill, st);
    alloc_n<int>(crow, nfill, st);
    alloc_n<int>(ccol, nfill, st);
    alloc_n<int>(sidx, nfill, st);
    k_p0_schur_emit<<<nblk(p), TPB, 0, st>>>(p, dp.cell_nbr_off.as<int64_t>(), poff.as<int64_t>(),
                                              dp.cell_nbr.as<int>(), dp.cell_nbr_col.as<int>(), uoff.as<int64_t>(),
                                              dp.bh.as<int>(), sk.as<unsigned long long>(), crow.as<int>(),
                                              ccol.as<int>(), sidx.as<int>());
    L();
    alloc_n<unsigned long long>(sks, nfill, st);
    alloc_n<int>(sidx2, nfill, st);
    size_t b = 0;
    GCK(cub::DeviceRadixSort::SortPairs(nullptr, b, sk.as<unsigned long long>(), sks.as<unsigned long long>(),
                                        sidx.as<int>(), sidx2.as<int>(), nfill, 0, 64, st));
    GCK(cub::DeviceRadixSort::SortPairs(tmp.get(b), b, sk.as<unsigned long long>(), sks.as<unsigned long long>(),
                                        sidx.as<int>(), sidx2.as<int>(), nfill, 0, 64, st));
    alloc_n<int>(dp.con_cell, nfill, st);
    alloc_n<int>(dp.con_row, nfill, st);
    alloc_n<int>(dp.con_col, nfill, st);
    alloc_n<int>(hd, nfill, st);
    alloc_n<int>(sg, nfill, st);
    k_p0_schur_out<<<nblk(nfill), TPB, 0, st>>>(sks.as<unsigned long long>(), sidx2.as<int>(), crow.as<int>(),
                                                 ccol.as<int>(), nfill, dp.con_cell.as<int>(), dp.con_row.as<int>(),
                                                 dp.con_col.as<int>(), hd.as<int>());
    L();
    scan_incl(hd.as<int>(), sg.as<int>(), nfill, tmp, st);
    const int ntgt = nfill ? read1(sg.as<int>() + nfill - 1, st) : 0;
    alloc_n<int>(dp.tgt_blk, ntgt, st);
    alloc_n<int64_t>(dp.tgt_off, ntgt + 1, st);
    GCK(cudaMemsetAsync(dp.tgt_off.p, 0, sizeof(int64_t), st));
    if (nfill) {
      k_p0_tgt<<<nblk(nfill), TPB, 0, st>>>(sks.as<unsigned long long>(), sg.as<int>(), hd.as<int>(), nfill,
                                             dp.tgt_blk.as<int>(), dp.tgt_off.as<int64_t>());
      L();
    }
    dp.ntgt = ntgt;
    lap("schur targets");
  }
  // ---- block Jacobi scaling blocks, skeleton lists --------------------------------------------
  const int nscale = select_idx(fscale.as<uint8_t>(), (int)nb, dp.scale_blk, tmp, cnt, st);
  DBuf sk_index, skn, sks_cnt, sk_soff;
  alloc_n<int>(sk_index, G, st);
  GCK(cudaMemsetAsync(sk_index.p, 0xff, (size_t)G * sizeof(int), st));
  k_p0_sk_index<<<nblk(nsk), TPB, 0, st>>>(dp.skeleton.as<int>(), nsk, sk_index.as<int>());
  L();
  alloc_n<int64_t>(skn, nsk, st);
  alloc_n<int64_t>(sks_cnt, nsk, st);
  alloc_n<int>(dp.sk_ndep, nsk, st);
  k_p0_sk_counts<<<nblk(nsk), TPB, 0, st>>>(dp.skeleton.as<int>(), nsk, dp.adj_off.as<int64_t>(),
                                             dp.adj_nbr.as<int>(), dp.kind.as<int>(), sk_index.as<int>(),
                                             skn.as<int64_t>(), dp.sk_ndep.as<int>(), sks_cnt.as<int64_t>());
  L();
  const int64_t nskn = offsets(skn, dp.sk_nbr_off, nsk, tmp, st);
  const int64_t nsucc = offsets(sks_cnt, dp.sk_succ_off, nsk, tmp, st);
  alloc_n<int>(dp.sk_nbr, nskn, st);
  alloc_n<int>(dp.sk_nbr_blk, nskn, st);
  alloc_n<int>(dp.sk_succ, nsucc, st);
  k_p0_sk_fill<<<nblk(nsk), TPB, 0, st>>>(dp.skeleton.as<int>(), nsk, dp.adj_off.as<int64_t>(), dp.adj_nbr.as<int>(),
                                           dp.adj_blk.as<int>(), dp.kind.as<int>(), sk_index.as<int>(),
                                           dp.sk_nbr_off.as<int64_t>(), dp.sk_succ_off.as<int64_t>(),
                                           dp.sk_nbr.as<int>(), dp.sk_nbr_blk.as<int>(), dp.sk_succ.as<int>());
  L();
  GCK(cudaGetLastError());
  const int badv = read1(bad.as<int>(), st);
  if (badv == 2) throw std::runtime_error("planner: two interior groups coupled");
  if (badv == 1 || badv == 3) throw std::runtime_error("planner: interior group is not first in its closure");
  g_launches.fetch_add(nlaunch, std::memory_order_relaxed);
  lap("skeleton lists");
  // ---- host copies of what the level loop reads ------------------------------------------------
  // one batched transfer: every array into one pinned staging buffer (one synchronisation), then a
  // single parallel copy-out into recycled (already faulted-in) host vectors
  Groups& g = lp.grp;
  g.level = 0;
  g.G = G;
  std::vector<int> hkey;
  {
    struct Item {
      void* host;
      const void* dev;
      size_t bytes;
    };
    std::vector<Item> items;
    auto want_i = [&](std::vector<int>& h, const DBuf& d, int64_t n) {
      pool_take(h, n);
      if (n) items.push_back({h.data(), d.p, (size_t)n * sizeof(int)});
    };
    auto want_l = [&](std::vector<int64_t>& h, const DBuf& d, int64_t n) {
      pool_take(h, n);
      if (n) items.push_back({h.data(), d.p, (size_t)n * sizeof(int64_t)});
    };
    want_l(g.off, dp.goff, G + 1);
    want_i(g.mem, dp.mem, N);
    want_i(g.kind, dp.kind, G);
    want_i(hkey, gkey, G);
    want_i(lp.pat.bg, dp.bg, nb);
    want_i(lp.pat.bh, dp.bh, nb);
    want_i(lp.interior, dp.interior, p);
    want_i(lp.precond, dp.precond, r);
    want_i(lp.skeleton, dp.skeleton, nsk);
    want_l(lp.cell_nbr_off, dp.cell_nbr_off, p + 1);
    want_i(lp.cell_nbr, dp.cell_nbr, ncn);
    want_i(lp.cell_n, dp.cell_n, p);
    want_i(lp.cell_b, dp.cell_b, p);
    want_i(lp.tgt_blk, dp.tgt_blk, dp.ntgt);
    want_i(lp.scale_blk, dp.scale_blk, nscale);
    want_l(lp.sk_nbr_off, dp.sk_nbr_off, nsk + 1);
    want_i(lp.sk_nbr, dp.sk_nbr, nskn);
    size_t tot = 0;
    for (auto& it : items) tot += (it.bytes + 255) & ~size_t(255);
    static char* pin = nullptr;
    static size_t pin_cap = 0;
    static std::mutex pin_mu;
    std::lock_guard<std::mutex> lock(pin_mu);
    if (tot > pin_cap) {
      if (pin) cudaFreeHost(pin);
      pin_cap = tot + (tot >> 2);
      if (cudaHostAlloc((void**)&pin, pin_cap, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        pin = nullptr;
        pin_cap = 0;
      }
    }
    if (pin) {
      size_t o = 0;
      std::vector<size_t> at(items.size());
      for (size_t q = 0; q < items.size(); ++q) {
        at[q] = o;
        GCK(cudaMemcpyAsync(pin + o, items[q].dev, items[q].bytes, cudaMemcpyDeviceToHost, st));
        o += (items[q].bytes + 255) & ~size_t(255);
      }
      GCK(cudaStreamSynchronize(st));
      // chunks of <= 1 MB over all arrays, copied out in parallel
      std::vector<std::tuple<size_t, size_t, size_t>> chunks;   // (item, offset, length)
      for (size_t q = 0; q < items.size(); ++q)
        for (size_t a0 = 0; a0 < items[q].bytes; a0 += (size_t)1 << 20)
          chunks.emplace_back(q, a0, std::min<size_t>((size_t)1 << 20, items[q].bytes - a0));
#pragma omp parallel for schedule(dynamic, 1)
      for (int64_t c = 0; c < (int64_t)chunks.size(); ++c) {
        const auto& ck = chunks[c];
        const size_t q = std::get<0>(ck), a0 = std::get<1>(ck), len = std::get<2>(ck);
        memcpy(static_cast<char*>(items[q].host) + a0, pin + at[q] + a0, len);
      }
    } else {
      for (auto& it : items) download_bytes(it.host, it.dev, it.bytes, st);
    }
  }
  g.q.assign(3 * (size_t)G, 0);
  g.bits.assign(G, 0);
  for (int i = 0; i < G; ++i) {
    g.bits[i] = hkey[i] & ((1 << dim) - 1);
    int64_t k = hkey[i] >> dim;
    for (int d = dim - 1; d >= 0; --d) {
      g.q[3 * i + d] = (int)(k % per);
      k /= per;
    }
  }
  lp.level = 0;
  lp.root = s.L == 0;
  lap("downloads");
  dp.nblocks = nb;
  dp.ncon = nfill;
  dp.nscale = nscale;
  dp.nsk_nbr = nskn;
  dp.nsucc = nsucc;
  // (the dependency wavefronts are formed later by the engine, off the critical path:
  // compute_waves, while the GPU eliminates the level's cells)
  dp.valid = true;
}

// full download (for the planner check): every array the host planner produces
void download_plan0(DevPlan0& dp, LevelPlan& lp, cudaStream_t st) {
  const int G = lp.grp.G, p = (int)lp.interior.size(), nsk = (int)lp.skeleton.size();
  down(lp.pat.adj_off, dp.adj_off, G + 1, st);
  const int64_t nadj = lp.pat.adj_off.empty() ? 0 : lp.pat.adj_off[G];
  down(lp.pat.adj_nbr, dp.adj_nbr, nadj, st);
  down(lp.pat.adj_blk, dp.adj_blk, nadj, st);
  down(lp.boff, dp.boff, dp.nblocks, st);
  const int64_t ncn = lp.cell_nbr_off.empty() ? 0 : lp.cell_nbr_off[p];
  down(lp.cell_nbr_blk, dp.cell_nbr_blk, ncn, st);
  down(lp.cell_nbr_col, dp.cell_nbr_col, ncn, st);
  down(lp.tgt_off, dp.tgt_off, dp.ntgt + 1, st);
  down(lp.con_cell, dp.con_cell, dp.ncon, st);
  down(lp.con_row, dp.con_row, dp.ncon, st);
  down(lp.con_col, dp.con_col, dp.ncon, st);
  down(lp.sk_nbr_blk, dp.sk_nbr_blk, dp.nsk_nbr, st);
  down(lp.sk_ndep, dp.sk_ndep, nsk, st);
  down(lp.sk_succ_off, dp.sk_succ_off, nsk + 1, st);
  down(lp.sk_succ, dp.sk_succ, dp.nsucc, st);
}

}  // namespace phif
