// Host driver of the B200 PHIF engine (CUDA runtime; one handle per factorization).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>
#include <stdexcept>
#include <string>
#include <future>
#include <vector>

#include "launch.h"
#include "planner.h"

namespace phif {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct NotSpd : std::runtime_error {
  int pivot, level, stage, group;
  std::string partial;   // stats JSON of the levels completed before the failure
  NotSpd(int p, int l, int s, int g)
      : std::runtime_error("not SPD"), pivot(p), level(l), stage(s), group(g) {}
};

enum Stage { ST_ELIMINATE = 0, ST_PRECONDITION = 1, ST_SKELETONIZE = 2, ST_ROOT = 3 };

// Device allocation owned by a handle (stream-ordered).
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t s = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept { *this = std::move(o); }
  DBuf& operator=(DBuf&& o) noexcept;
  ~DBuf() { release(); }
  void alloc(size_t nbytes, cudaStream_t st, bool zero = false);
  void release();
  template <class T>
  T* as() const { return reinterpret_cast<T*>(p); }
};

// host -> device copy on stream s; large copies go through a pinned staging ring (engine.cu)
void upload_bytes(void* dst, const void* src, size_t bytes, cudaStream_t s);
// device -> host copy through pinned staging (synchronises the stream)
void download_bytes(void* dst, const void* src, size_t bytes, cudaStream_t s);
template <class T>
void upload(DBuf& b, const std::vector<T>& v, cudaStream_t s) {
  b.alloc(std::max<size_t>(1, v.size()) * sizeof(T), s);
  if (!v.empty()) upload_bytes(b.p, v.data(), v.size() * sizeof(T), s);
}

struct Matrix {
  int64_t N = 0, nnz = 0;
  // assembled on the device from a coefficient field (problem.cu): the field and the diagonal
  // are kept for the matrix-free stencil SpMV
  bool stencil = false;
  int dim = 0;
  int64_t side = 0;
  DBuf field, diag;
  // host copy of the pattern for the host planner (uninitialised allocations filled by parallel
  // copies; downloaded on first use for a matrix assembled on the device)
  mutable std::unique_ptr<int64_t[]> h_rowptr;
  mutable std::unique_ptr<int[]> h_col;
  void ensure_host_pattern(cudaStream_t s) const;
  DBuf rowptr, col, val;
};

struct BigApply;   // GEMM replay of big records (engine.cu)

struct BdLists {
  std::vector<int> dof;
  std::vector<int64_t> off;
  std::vector<int> rows;
};

struct LevelRT {
  LevelPlan plan;
  ~LevelRT() { recycle_plan(plan); }
  // structure on device
  DBuf goff, mem, gsize, boff, bg, bh, adj_off, adj_nbr, adj_blk, diag_blk;
  DBuf pool;   // live matrix blocks (freed after the level transition)
  DBuf rec;    // factor records of this level (persist)
  int64_t rec_doubles = 0;
  // cells
  DBuf c_interior, c_nbr_off, c_nbr_blk, c_nbr_col, c_nbr_w, c_n, c_b, c_P_off, c_U_off;
  DBuf c_I_off, c_B, c_B_off, c_work_off;
  DBuf bd_dof, bd_off, bd_rows;
  std::future<BdLists> bd_task;   // built on a host thread during the factorization
  std::vector<int> h_small_cells, h_big_cells;
  std::vector<int64_t> h_P_off, h_I_off, h_B_off, h_cwork;
  DBuf d_small_cells;
  std::shared_ptr<BigApply> bigap;
  int nbd = 0;
  int64_t cell_work_unit = 0, wbuf_unit = 0;
  // precondition
  DBuf p_groups, p_L_off, p_L_off_of_group, p_scale_blk, p_n, p_I_off, p_work_off;
  DBuf d_prec_small, d_scale_small;
  std::vector<int> h_prec_big;
  std::vector<int64_t> h_L_off, h_pI_off, h_pwork, h_T_off, h_SP_off, h_awork, h_S_off, h_R_off;
  std::vector<int> h_pn, h_sr, h_skt;
  DBuf d_apply_small_sk, d_apply_small_pr;
  int n_apply_small_sk = 0, n_apply_small_pr = 0;
  int cell_nmax = 0, cell_bmax = 0;   // largest cell of the level (picks the warp-per-cell replay)
  int n_apply_tiny_sk = 0, apply_tiny_rows = 1, apply_small_pr_max = 1;   // separators replayed one warp each
  DBuf d_apply_tiny_sk;
  std::shared_ptr<struct GemmReplay> replay;
  int64_t prec_work_unit = 0;
  // skeleton
  DBuf s_groups, s_nbr_off, s_nbr, s_nbr_blk, s_order, s_rank, s_T_off, s_P_off, s_work_off, s_iwork_off;
  DBuf s_r, s_kt, s_S, s_S_off, s_R, s_R_off, s_awork_off;
  std::vector<int> h_rank;
  int64_t skel_work_unit = 0;
  // stats
  double t_ms[6] = {0, 0, 0, 0, 0, 0};   // repack, eliminate, precondition, id, skel update, host plan
  double t_wall_ms = 0;
  double t_host_overlap_ms = 0;   // host descriptor work done while the GPU runs this level
  // algorithmic work per stage (0 repack, 1 eliminate+schur, 2 precondition, 3 id, 4 skel update)
  double fl[6] = {0, 0, 0, 0, 0, 0}, by[6] = {0, 0, 0, 0, 0, 0};
  DBuf s_rows;
  int rho_max = 0;
  double rho_mean = 0.0;
  double sep_k_mean = 0, sep_k_max = 0, sep_m_mean = 0, sep_m_max = 0, team_P_mean = 0;
  int n_large = 0;
  int n_gid = 0;      // separators on the Gram-path ID
  int64_t S = 0;
  LevelDev dev() const;
  // apply descriptors of the separators (built on a host thread; declared last so that it is
  // joined before the members it fills are destroyed)
  std::future<void> ap_task;
};

struct Factorization {
  Spec spec;
  int method = 1;  // 0 hif, 1 phif, 2 exact
  double eps = 0.0;
  cudaStream_t stream = 0;
  std::vector<std::unique_ptr<LevelRT>> levels;
  DBuf alive, red, status;
  DBuf work, wbuf;   // apply workspaces (sized for the largest nrhs seen)
  size_t work_cap = 0, wbuf_cap = 0;
  int64_t rec_bytes = 0;
  double t_factor_ms = 0.0, t_plan_ms = 0.0;
  std::string stats_json() const;
};

std::unique_ptr<Matrix> matrix_create(const int64_t* rowptr, const int* col, const double* val, int64_t N,
                                      cudaStream_t s);
std::unique_ptr<Factorization> factorize(const Matrix& A, int dim, int n, int m, double eps, int method,
                                         cudaStream_t s, bool timing);
// x (device, N x k row-major) transformed in place; mode 0 = F^-1, 1 = G^-1, 2 = G^-T
void apply(Factorization& F, double* x, int k, int mode);
struct PcgResult {
  std::vector<int> iters;
  std::vector<double> relres;
  std::vector<int> converged;
  std::vector<double> history;   // history_len x k relative residuals (row per iteration)
  int history_len = 0;
  int breakdown = 0;
};
PcgResult pcg(const Matrix& A, Factorization* F, const double* b, double* x, int k, double tol, int maxit,
              cudaStream_t s, bool want_history = false);
struct PowerResult {
  double value = 0.0;
  int iters = 0;
  int converged = 0;
  double rel = 0.0;
};
// e_s: power iteration on x -> x - G^-1 A G^-T x from the start vector x0 (host, length N)
PowerResult solve_error(const Matrix& A, Factorization& F, const double* x0, double rel_tol, int maxit);
// e_a = ||A - F|| / ||A|| by two power iterations from x0
PowerResult apply_error(const Matrix& A, Factorization& F, const double* x0, double rel_tol, int maxit);
// copy the root Cholesky factor B_L (row-major lower, n x n) to out (host or device; NULL: size only); returns n
int root_factor(Factorization& F, double* out);

}  // namespace phif
