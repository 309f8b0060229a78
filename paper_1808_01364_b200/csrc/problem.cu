// On-device problem generation and ingest.
//
// * Gaussian smoothing of a host-drawn white-noise / uniform lattice (the numpy PCG64 draws stay
//   on the host, default_rng(seed)): separable correlations along each axis in order, "reflect"
//   boundary, truncate 4, restating scipy.ndimage.gaussian_filter (the reference's generate_field,
//   grid.py:182-210) with its symmetric-kernel summation order -- center tap first, then
//   (x[i-j] + x[i+j]) * w[j] from the outermost tap inward, no fused multiply-add -- so the
//   smoothed field is bit-identical to the host one; then the threshold a = g > 0 ? hi : lo.
// * Stencil assembly of -div(a grad u) + b u (grid.py:213-260) straight into the device CSR:
//   arithmetic-mean fluxes, h^2 scaling, the diagonal accumulated in the reference's order
//   (b h^2, then per axis: the flux to the upper neighbour, the flux from the lower neighbour,
//   the two Dirichlet boundary terms), so the CSR equals the host assemble_operator's bit for bit.
// * Matrix-free stencil SpMV (grid.py:157-158): the off-diagonal values recomputed from the field
//   per edge, the diagonal stored; same terms, same order, same FMAs as the CSR SpMV.
#include <cub/cub.cuh>

#include <atomic>
#include <string>

#include "engine.h"
#include "problem.h"

namespace phif {

extern std::atomic<long long> g_launches;

namespace {

#define PCK(x)                                                                                   \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess) throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));    \
  } while (0)

__device__ __forceinline__ int64_t reflect_idx(int64_t i, int64_t len) {
  // scipy "reflect" (d c b a | a b c d | d c b a), any distance
  const int64_t per = 2 * len;
  int64_t m = i % per;
  if (m < 0) m += per;
  return m < len ? m : per - 1 - m;
}

// one correlation along `axis` of an (n0, n1, n2) Fortran-ordered lattice (x fastest)
__global__ void k_gauss_axis(const double* in, double* out, int64_t n0, int64_t n1, int64_t n2, int axis,
                             const double* w, int r) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t tot = n0 * n1 * n2;
  if (e >= tot) return;
  const int64_t c0 = e % n0, c1 = (e / n0) % n1, c2 = e / (n0 * n1);
  int64_t len, stride, pos;
  if (axis == 0) {
    len = n0, stride = 1, pos = c0;
  } else if (axis == 1) {
    len = n1, stride = n0, pos = c1;
  } else {
    len = n2, stride = n0 * n1, pos = c2;
  }
  const double* line = in + (e - pos * stride);
  double acc = __dmul_rn(line[pos * stride], w[r]);
  for (int j = r; j >= 1; --j) {
    const double lo = line[reflect_idx(pos - j, len) * stride];
    const double hi = line[reflect_idx(pos + j, len) * stride];
    acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(lo, hi), w[r - j]));
  }
  out[e] = acc;
}

__global__ void k_threshold(double* a, int64_t n, double lo, double hi) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) a[e] = a[e] > 0.0 ? hi : lo;
}

struct Grid3 {
  int dim;
  int64_t side;
  __device__ void coords(int64_t r, int64_t c[3]) const {
    c[0] = r % side;
    c[1] = dim > 1 ? (r / side) % side : 0;
    c[2] = dim > 2 ? r / (side * side) : 0;
  }
  __device__ int64_t stride(int d) const { return d == 0 ? 1 : (d == 1 ? side : side * side); }
};

__device__ __forceinline__ double flux(const double* a, int64_t p, int64_t q) {
  return __dmul_rn(0.5, __dadd_rn(a[p], a[q]));
}

__global__ void k_row_count(Grid3 g, int64_t N, int64_t* cnt) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= N) return;
  int64_t c[3];
  g.coords(r, c);
  int64_t k = 1;
  for (int d = 0; d < g.dim; ++d) k += (c[d] > 0) + (c[d] < g.side - 1);
  cnt[r] = k;
}

__global__ void k_diag(Grid3 g, int64_t N, const double* a, double bh2, double* diag) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= N) return;
  int64_t c[3];
  g.coords(r, c);
  double s = bh2;
  for (int d = 0; d < g.dim; ++d) {
    const int64_t st = g.stride(d);
    if (c[d] < g.side - 1) s = __dadd_rn(s, flux(a, r, r + st));   // diag[lo] += flux
    if (c[d] > 0) s = __dadd_rn(s, flux(a, r - st, r));             // diag[hi] += flux
    if (c[d] == 0) s = __dadd_rn(s, a[r]);                          // first boundary
    if (c[d] == g.side - 1) s = __dadd_rn(s, a[r]);                 // last boundary
  }
  diag[r] = s;
}

__global__ void k_fill_csr(Grid3 g, int64_t N, const double* a, const double* diag, const int64_t* rowptr, int* col,
                           double* val) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= N) return;
  int64_t c[3];
  g.coords(r, c);
  int64_t o = rowptr[r];
  for (int d = g.dim - 1; d >= 0; --d)   // lower neighbours, ascending column
    if (c[d] > 0) {
      const int64_t q = r - g.stride(d);
      col[o] = (int)q;
      val[o++] = -flux(a, q, r);
    }
  col[o] = (int)r;
  val[o++] = diag[r];
  for (int d = 0; d < g.dim; ++d)   // upper neighbours, ascending column
    if (c[d] < g.side - 1) {
      const int64_t q = r + g.stride(d);
      col[o] = (int)q;
      val[o++] = -flux(a, r, q);
    }
}

// y = A x for k right-hand sides (row-major N x k), entries in CSR order (ascending column)
__global__ void k_spmv_stencil(Grid3 g, int64_t N, const double* a, const double* diag, const double* x, double* y,
                               int k) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= N * k) return;
  const int64_t r = e / k;
  const int cc = (int)(e % k);
  int64_t c[3];
  g.coords(r, c);
  double s = 0.0;
  for (int d = g.dim - 1; d >= 0; --d)
    if (c[d] > 0) {
      const int64_t q = r - g.stride(d);
      s = __fma_rn(-flux(a, q, r), x[q * k + cc], s);
    }
  s = __fma_rn(diag[r], x[r * k + cc], s);
  for (int d = 0; d < g.dim; ++d)
    if (c[d] < g.side - 1) {
      const int64_t q = r + g.stride(d);
      s = __fma_rn(-flux(a, r, q), x[q * k + cc], s);
    }
  y[e] = s;
}

inline unsigned nb(int64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace

void smooth_field(int dim, int64_t side, double* d_field, const std::vector<double>& weights, cudaStream_t s) {
  const int r = (int)(weights.size() / 2);
  const int64_t n0 = side, n1 = dim > 1 ? side : 1, n2 = dim > 2 ? side : 1, N = n0 * n1 * n2;
  DBuf w, tmp;
  w.alloc(weights.size() * sizeof(double), s);
  PCK(cudaMemcpyAsync(w.p, weights.data(), weights.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  tmp.alloc(N * sizeof(double), s);
  double* src = d_field;
  double* dst = tmp.as<double>();
  for (int ax = 0; ax < dim; ++ax) {
    k_gauss_axis<<<nb(N), 256, 0, s>>>(src, dst, n0, n1, n2, ax, w.as<double>(), r);
    std::swap(src, dst);
  }
  if (src != d_field) PCK(cudaMemcpyAsync(d_field, src, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
  g_launches.fetch_add(dim, std::memory_order_relaxed);
}

void threshold_field(double* d_field, int64_t N, double lo, double hi, cudaStream_t s) {
  k_threshold<<<nb(N), 256, 0, s>>>(d_field, N, lo, hi);
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

std::unique_ptr<Matrix> matrix_from_field(int dim, int n, const double* d_field, double bh2, cudaStream_t s,
                                          bool host_pattern) {
  auto A = std::make_unique<Matrix>();
  Grid3 g{dim, n - 1};
  int64_t N = 1;
  for (int d = 0; d < dim; ++d) N *= (n - 1);
  A->N = N;
  A->stencil = true;
  A->dim = dim;
  A->side = n - 1;
  A->field.alloc(N * sizeof(double), s);
  PCK(cudaMemcpyAsync(A->field.p, d_field, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
  A->diag.alloc(N * sizeof(double), s);
  k_diag<<<nb(N), 256, 0, s>>>(g, N, A->field.as<double>(), bh2, A->diag.as<double>());
  DBuf cnt;
  cnt.alloc(N * sizeof(int64_t), s);
  k_row_count<<<nb(N), 256, 0, s>>>(g, N, cnt.as<int64_t>());
  A->rowptr.alloc((N + 1) * sizeof(int64_t), s);
  PCK(cudaMemsetAsync(A->rowptr.p, 0, sizeof(int64_t), s));
  {
    size_t b = 0;
    PCK(cub::DeviceScan::InclusiveSum(nullptr, b, cnt.as<int64_t>(), A->rowptr.as<int64_t>() + 1, N, s));
    DBuf tmp;
    tmp.alloc(b, s);
    PCK(cub::DeviceScan::InclusiveSum(tmp.p, b, cnt.as<int64_t>(), A->rowptr.as<int64_t>() + 1, N, s));
  }
  int64_t nnz = 0;
  PCK(cudaMemcpyAsync(&nnz, A->rowptr.as<int64_t>() + N, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  PCK(cudaStreamSynchronize(s));
  A->nnz = nnz;
  A->col.alloc(nnz * sizeof(int), s);
  A->val.alloc(nnz * sizeof(double), s);
  k_fill_csr<<<nb(N), 256, 0, s>>>(g, N, A->field.as<double>(), A->diag.as<double>(), A->rowptr.as<int64_t>(),
                                    A->col.as<int>(), A->val.as<double>());
  g_launches.fetch_add(3, std::memory_order_relaxed);
  if (host_pattern) {   // (the host planner path needs the pattern on the host)
    A->h_rowptr.reset(new int64_t[N + 1]);
    A->h_col.reset(new int[std::max<int64_t>(nnz, 1)]);
    download_bytes(A->h_rowptr.get(), A->rowptr.p, (N + 1) * sizeof(int64_t), s);
    download_bytes(A->h_col.get(), A->col.p, nnz * sizeof(int), s);
  }
  PCK(cudaStreamSynchronize(s));
  PCK(cudaGetLastError());
  return A;
}

void spmv(const Matrix& A, const double* x, double* y, int k, cudaStream_t s) {
  if (A.stencil && !getenv("PHIF_CSR_SPMV")) {
    Grid3 g{A.dim, A.side};
    k_spmv_stencil<<<nb(A.N * k), 256, 0, s>>>(g, A.N, A.field.as<double>(), A.diag.as<double>(), x, y, k);
    g_launches.fetch_add(1, std::memory_order_relaxed);
  } else {
    launch_spmv(A.rowptr.as<int64_t>(), A.col.as<int>(), A.val.as<double>(), x, y, A.N, k, s);
  }
}

}  // namespace phif
