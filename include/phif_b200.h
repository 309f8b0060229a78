/*
 * phif_b200.h - C-ABI of the B200-native PHIF (arXiv 1808.01364) engine.
 *
 * The reference (pkg/src/hifsolve, Python) specifies its hot path as Python
 * functions in modules that are absent from the tree. Each
 * entry point below is what a ctypes / cffi binding of that Python API binds
 * (see INTEGRATION.md); the Python mirror lives in paper_1808_01364_b200/.
 *
 *   reference interface (file:line)                  -> C entry point
 *   SymSparseMatrix(csr)          grid.py:124-147    -> phif_matrix_create
 *   factorize(A, spec, eps, method) SPEC.md:275-283  -> phif_factorize
 *   apply_inverse(Fz, b)          SPEC.md:293-301    -> phif_apply(mode 0)
 *   apply_ginv(Fz, x)             SPEC.md:302-306    -> phif_apply(mode 1)
 *   apply_ginv_t(Fz, x)           SPEC.md:302-306    -> phif_apply(mode 2)
 *   apply(Fz, x)  (F x)           SPEC.md:284-292    -> phif_apply(mode 3)
 *   pcg(A, b, precond, tol, maxit) SPEC.md:360-378   -> phif_pcg
 *   estimate_solve_error(A, Fz)   SPEC.md:418-426    -> phif_solve_error
 *   estimate_apply_error(A, Fz)   SPEC.md:409-417    -> phif_apply_error
 *   root_condition(Fz)            SPEC.md:311-319    -> phif_root_factor (+ host SVD)
 *   Factorization stats JSON      SPEC.md:341        -> phif_stats_json
 *   skeleton sets of the records  SPEC.md:235        -> phif_skeleton_sets
 *   classify_active(spec, l, S)   hierarchy.py:102   -> phif_classify
 *
 * Conventions: no exception crosses the boundary; every function returns an
 * int status (PHIF_OK, PHIF_NOT_SPD, PHIF_BREAKDOWN, PHIF_ERROR). NotSpd carries
 * (pivot 0-based as kernels.py:32, level, stage, group) like errors.py:21-30.
 * Vector arguments may be host or device pointers (detected); vectors with
 * nrhs columns are N x nrhs row-major (DOF-major). `stream` is a cudaStream_t.
 * A finished factor is read-only and safe for concurrent callers: apply / pcg /
 * estimator calls on one factor from several host threads are serialised per factor (each call
 * is synchronous), calls on different factors run concurrently.
 */
#ifndef PHIF_B200_H
#define PHIF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PHIF_OK 0
#define PHIF_ERROR 1
#define PHIF_NOT_SPD 2
#define PHIF_BREAKDOWN 3

#define PHIF_METHOD_HIF 0
#define PHIF_METHOD_PHIF 1
#define PHIF_METHOD_EXACT 2

#define PHIF_STAGE_ELIMINATE 0
#define PHIF_STAGE_PRECONDITION 1
#define PHIF_STAGE_SKELETONIZE 2
#define PHIF_STAGE_ROOT 3

typedef struct phif_matrix phif_matrix;
typedef struct phif_factor phif_factor;

typedef struct phif_error {
  int code;
  int pivot;
  int level;
  int stage;
  int group;
  char message[512];
} phif_error;

int phif_version(void);

/* Number of engine kernel launches issued so far in this process (evidence counter). */
long long phif_launch_count(void);

/* Symmetric CSR (full pattern, sorted columns) from host arrays; uploaded to HBM. */
int phif_matrix_create(const int64_t* rowptr, const int32_t* col, const double* val, int64_t n, void* stream,
                       phif_matrix** out, phif_error* err);
void phif_matrix_free(phif_matrix* A);

/* On-device problem generation and assembly (grid.py:182-260): the nodal
 * coefficient lattice a ((n-1)^dim values, x fastest; host or device pointer) is Gaussian-smoothed
 * on the device with the given symmetric weights (scipy.ndimage.gaussian_filter order, reflect
 * boundary; nweights = 0: none), thresholded to a > 0 ? hi : lo (lo = hi = 0: none), and A =
 * -div(a grad u) + b u is assembled on the device (bh2 = b h^2) bit-identically to
 * assemble_operator. The matrix keeps the field for the matrix-free stencil SpMV that phif_pcg and
 * the estimators then use. */
int phif_matrix_from_field(int dim, int n, const double* a, const double* weights, int nweights, double lo, double hi,
                           double bh2, void* stream, phif_matrix** out, phif_error* err);

/* Copy A to host arrays (any output may be NULL): *nnz, rowptr (N+1), col, val (nnz), and the
 * coefficient field (N) of a matrix built by phif_matrix_from_field. */
int phif_matrix_csr(const phif_matrix* A, int64_t* nnz, int64_t* rowptr, int32_t* col, double* val, double* field);

/* y = A x for host arrays (N x nrhs): the engine's SpMV (matrix-free stencil when A carries its
 * field, unless force_csr). */
int phif_matrix_apply(const phif_matrix* A, const double* x, double* y, int nrhs, int force_csr, phif_error* err);

/* factorize(A, GridSpec(dim, n, m), eps, method); timing != 0 records per-stage CUDA events. */
int phif_factorize(const phif_matrix* A, int dim, int n, int m, double eps, int method, void* stream, int timing,
                   phif_factor** out, phif_error* err);
void phif_factor_free(phif_factor* F);

/* x <- op(F) x in place, op: 0 = F^-1 (apply_inverse), 1 = G^-1, 2 = G^-T,
 * 3 = F (apply), 4 = G^T, 5 = G. x: N x nrhs, host or device. */
int phif_apply(phif_factor* F, double* x, int nrhs, int mode, phif_error* err);

/* PCG with F^-1 (F may be NULL for plain CG). b, x: N x nrhs. Per column outputs. history (may be
 * NULL) receives the relative residual of every column after every iteration (row-major,
 * iteration x nrhs, room for maxit rows: SolveReport residual history) and
 * *history_len the number of rows written. */
int phif_pcg(const phif_matrix* A, phif_factor* F, const double* b, double* x, int nrhs, double tol, int maxit,
             void* stream, int* iters, double* relres, int* converged, double* history, int* history_len,
             phif_error* err);

/* e_s = ||I - G^-1 A G^-T||_2 by power iteration from host start vector x0 (length N). */
int phif_solve_error(const phif_matrix* A, phif_factor* F, const double* x0, double rel_tol, int maxit,
                     double* value, int* iters, int* converged, double* rel_achieved, phif_error* err);

/* e_a = ||A - F||_2 / ||A||_2 by two power iterations from host start vector x0
 * (estimate_apply_error). */
int phif_apply_error(const phif_matrix* A, phif_factor* F, const double* x0, double rel_tol, int maxit,
                     double* value, int* iters, int* converged, double* rel_achieved, phif_error* err);

/* Root Cholesky factor B_L (|S_L| x |S_L| row-major lower) into out (host or device); out = NULL
 * only sets *n = |S_L|. Used by root_condition. */
int phif_root_factor(phif_factor* F, double* out, int* n, phif_error* err);

/* Statistics JSON; returns the length needed (excluding NUL), copies at most cap-1 bytes. */
size_t phif_stats_json(const phif_factor* F, char* buf, size_t cap);

/* Skeleton sets of level `level`: counts[0] = #skeleton groups, counts[1] = sum rank,
 * counts[2] = sum redundant. With non-NULL outputs also fills per group rank,
 * and redundant count, the skeleton DOFs and the redundant DOFs (ascending within each group, groups
 * in classify order). */
int phif_skeleton_sets(const phif_factor* F, int level, int64_t* counts, int32_t* rank, int32_t* nred,
                       int32_t* skel_dofs, int32_t* red_dofs);
int phif_num_levels(const phif_factor* F);

/* Statistics JSON of the levels a factorization completed before its last PHIF_NOT_SPD failure on
 * this thread (NotSpdError.partial_stats, errors.py:21-30 / SPEC.md:279); same contract as
 * phif_stats_json. */
size_t phif_last_partial_stats(char* buf, size_t cap);

/* Planner check (CPU only): group the active DOFs of `level` like classify_active.
 * group_of[i] = group index (classify order) of active[i]; kind_of_group[g] = number of
 * on-line axes. Returns the number of groups (or -1); kind_of_group may be NULL. */
int64_t phif_classify(int dim, int n, int m, int level, const int32_t* active, int64_t nactive, int32_t* group_of,
                      int32_t* kind_of_group, int64_t kind_cap);

/* Device planner check (GPU): plan level 0 of A's pattern on the host (planner.cpp) and on the
 * device (gpu_plan.cu, the level-0 planner factorize uses) and compare every plan array.
 * Returns the number of differing arrays (0 = identical, -1 = error); names them in `report`. */
int phif_plan_check(const phif_matrix* A, int dim, int n, int m, char* report, size_t cap);

/* Planner dry run (CPU only): plan every level of a factorization of the CSR pattern,
 * assuming the first `keep` DOFs of every separator group survive (keep < 0: all survive).
 * Writes one JSON object per level into buf (like phif_stats_json). */
size_t phif_plan_dryrun(int dim, int n, int m, const int64_t* rowptr, const int32_t* col, int keep, char* buf,
                        size_t cap);

#ifdef __cplusplus
}
#endif

#endif /* PHIF_B200_H */
