// On-device problem generation, stencil assembly and the matrix-free SpMV (problem.cu).
#pragma once
#include <memory>
#include <vector>

#include "engine.h"

namespace phif {

// Gaussian smoothing of a device lattice in place (scipy.ndimage.gaussian_filter order, reflect)
void smooth_field(int dim, int64_t side, double* d_field, const std::vector<double>& weights, cudaStream_t s);
// a <- a > 0 ? hi : lo
void threshold_field(double* d_field, int64_t N, double lo, double hi, cudaStream_t s);
// A = -div(a grad u) + b u (h^2-scaled) assembled on the device from the nodal field (copied in)
std::unique_ptr<Matrix> matrix_from_field(int dim, int n, const double* d_field, double bh2, cudaStream_t s,
                                          bool host_pattern);
// y = A x (k right-hand sides): matrix-free stencil when A carries its field, else CSR
void spmv(const Matrix& A, const double* x, double* y, int k, cudaStream_t s);

}  // namespace phif
