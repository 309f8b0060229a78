// Host-callable launch wrappers (implemented in kernels.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"

namespace phif {

struct ApplyCellArgs {
  int p;
  const int* list;   // cells replayed by the one-CTA kernel (nullptr = all)
  const int* n;
  const int* b;
  const int* I;
  const int64_t* I_off;
  const int* B;
  const int64_t* B_off;   // also the row offset of the cell's contribution inside wbuf
  const double* rec;
  const int64_t* P_off;
  double* work;
  const int64_t* work_off;  // (n+b) * k doubles per cell (scaled by k on the host)
  double* wbuf;
};

struct ApplyPrecArgs {
  int r;
  int ldn;           // largest group of the list (shared-memory staging of the warp kernel)
  const int* list;
  const int* n;
  const int* I;
  const int64_t* I_off;
  const double* rec;
  const int64_t* L_off;
  double* work;
  const int64_t* work_off;
};

struct ApplySkelArgs {
  int nsk;
  const int* list;
  const int* r;
  const int* kt;
  const int* S;
  const int64_t* S_off;
  const int* R;
  const int64_t* R_off;
  const double* rec;
  const int64_t* T_off;
  const int64_t* P_off;
  double* work;
  const int64_t* work_off;
};

void configure_kernels();
long long launch_count();   // kernel launches issued so far (all streams)
void launch_ingest(const LevelDev& lv, const int* gid, const int* pos, const int64_t* rowptr, const int* col,
                   const double* val, int64_t N, cudaStream_t s);
void launch_fill_int(int* p, int v, int64_t n, cudaStream_t s);
void launch_group_pos(const LevelDev& lv, int* gid, int* pos, cudaStream_t s);
void launch_cell(const LevelDev& lv, const CellArgs& a, int count, DevStatus* st, cudaStream_t s);
void launch_schur(const LevelDev& lv, const SchurArgs& a, cudaStream_t s);
void launch_prec_build(const LevelDev& lv, const PrecArgs& a, const int* list, int nbig, cudaStream_t s);
void launch_prec_factor(const LevelDev& lv, const PrecArgs& a, DevStatus* st, cudaStream_t s);
// gemm_only: every block of the list fits the two-GEMM form (|g| |h| <= 64 x 64)
void launch_prec_scale(const LevelDev& lv, const PrecArgs& a, cudaStream_t s, bool gemm_only = false);
void launch_prec_factor_warp(const LevelDev& lv, const PrecArgs& a, const int* list, int n, int kmax, DevStatus* st,
                             cudaStream_t s);
void launch_prec_scale_warp(const LevelDev& lv, const PrecArgs& a, const int* list, int n, int ldmax, cudaStream_t s);
void launch_skel_id(const LevelDev& lv, const SkelArgs& a, int count, int64_t need_doubles, cudaStream_t s);
// kmax: largest separator of the level (0 = unknown); picks the occupancy variant of the kernel
void launch_skel_id_dyn(const LevelDev& lv, const SkelArgs& a, const DynSched& ds, int64_t need_doubles,
                        cudaStream_t s, int kmax = 0);
int team_colcap(int vcap, int kmax);
int team_blocks_per_sm(int vcap, int kmax, int colcap);
void launch_skel_team(const LevelDev& lv, const SkelArgs& a, const TeamArgs& t, int nblocks, cudaStream_t s);
int team_max_clusters(int vcap, int kmax, int colcap, int csize);
// Gram-path ID: cluster size for separators up to kmax columns; *sg = Schur complement in global memory;
// *gbuf_doubles = workspace doubles per item of k columns (call with the item's k)
int gid_cluster(int kmax, bool* sg);
bool gid_fits(int k);
int64_t gid_gbuf_doubles(int k, int C, bool sg, int S);
void launch_gid(const LevelDev& lv, const SkelArgs& a, const GramArgs& g, int kmax, bool sg, cudaStream_t s);
int64_t gid_T_cap(int kmax);
void launch_gid_T(const LevelDev& lv, const SkelArgs& a, const GramArgs& g, int kmax, cudaStream_t s);
void launch_big_build(const LevelDev& lv, const CellArgs& ca, const int* big_cells, int nbig, cudaStream_t s);
void launch_big_step(const BigArgs& diag, const BigArgs& trsm, const BigArgs& upd, DevStatus* st, cudaStream_t s);
void launch_big_nt(const BigArgs& a, int mode, cudaStream_t s);
void launch_big_wide(const BigArgs& a, int mode, cudaStream_t s);   // 128 x 128 tiles
// banded level-0 cells (2D): shared-memory fit, the kernel, and the device band check
bool band_cells_fit(int nmax, int bmax, int w);
int64_t band_scratch_stride(int nmax, int w);   // doubles of one cell's band + reciprocals
void launch_cell_band(const LevelDev& lv, const CellArgs& ca, const int* list, int count, int nmax, int bmax, int w,
                      double* scratch, DevStatus* st, long long* prof, cudaStream_t s);
void launch_band_check(const int64_t* rowptr, const int* col, const int* gid, const int* pos, const uint8_t* is_int,
                       int64_t N, int w, int* flag, cudaStream_t s);
void launch_big_zero_upper(const BigArgs& a, cudaStream_t s);   // 0: trailing update, 1: U = X^T X
void launch_bgemm(const GemmDesc* desc, const int* w_desc, const int* w_tile, int nwork, cudaStream_t s);
// replay GEMM (N = nrhs <= 32, A streamed from global, B chunk in shared memory); falls back to launch_bgemm
// kmean: mean K depth per work item of this launch (picks the chunk depth of the kernel)
void launch_rgemm(const GemmDesc* desc, const int* w_desc, const int* w_tile, int nwork, int nrhs, cudaStream_t s,
                  int kmean = 0);
void launch_rows(double* Y, double* x, const int* idx, const int64_t* seg_src, const int64_t* seg_dst,
                 const int* seg_len, int nseg, int k, bool to_x, cudaStream_t s);
void launch_skel_update(const LevelDev& lv, const SkelArgs& a, const int* list, int count, DevStatus* st,
                        cudaStream_t s);
void launch_skel_big_gather(const LevelDev& lv, const SkelArgs& a, const int* big, const int* idx,
                            const int64_t* idx_off, int nbig, cudaStream_t s);
void launch_skel_big_post(const LevelDev& lv, const SkelArgs& a, const int* big, const int* idx, const int64_t* idx_off,
                          const double* U, const int64_t* U_off, int nbig, cudaStream_t s);
void launch_repack(const RepackArgs& a, cudaStream_t s);
void launch_apply_cell(const ApplyCellArgs& a, double* x, int k, bool up, cudaStream_t s);
// warp-per-cell DMMA replay of small cells (n <= 32, b <= 64) for 32 right-hand sides
bool apply_cell_mma_fits(int nmax, int bmax, int k);
void launch_apply_cell_mma(const ApplyCellArgs& a, int nmax, int bmax, double* x, bool up, cudaStream_t s);
void launch_apply_reduce(const int* dof, const int64_t* off, const int* rows, const double* wbuf, int nd, double* x,
                         int k, cudaStream_t s);
void launch_apply_prec(const ApplyPrecArgs& a, double* x, int k, bool up, cudaStream_t s);
void launch_apply_skel(const ApplySkelArgs& a, double* x, int k, bool up, cudaStream_t s);
void launch_apply_skel_warp(const ApplySkelArgs& a, const int* list, int n, double* x, int k, bool up, int ldrows,
                            cudaStream_t s);
// forward replay (F x = G G^T x): one CTA per cell / block-Jacobi group / separator record
void launch_fwd(const ApplyCellArgs* c, const ApplyPrecArgs* p, const ApplySkelArgs* sk, double* x, int k, bool up,
                cudaStream_t s);
void launch_spmv(const int64_t* rowptr, const int* col, const double* val, const double* x, double* y, int64_t N,
                 int k, cudaStream_t s);
int dot_part_blocks();
void launch_dot(const double* a, const double* b, int64_t N, int k, double* part, double* out, cudaStream_t s);
void launch_pcg_update(double* x, const double* p, double* r, const double* q, const double* alpha, const int* active,
                       int64_t N, int k, double* part, double* rn2, cudaStream_t s);
void launch_axpy(double* y, const double* x, const double* coef, double sgn, const int* active, int64_t N, int k,
                 cudaStream_t s);
void launch_xpby(double* p, const double* z, const double* coef, const int* active, int64_t N, int k,
                 cudaStream_t s);
void launch_sub(double* r, const double* b, const double* q, const int* active, int64_t N, int k, cudaStream_t s);
void launch_pcg_init(const double* bn2, double* bn, int* active, double* relres, int* iters, int* conv, int* ctl,
                     int k, cudaStream_t s);
void launch_pcg_alpha(const double* rz, const double* pq, const int* active, double* alpha, int* ctl, int it, int k,
                      cudaStream_t s);
void launch_pcg_check(const double* rn2, const double* bn, int* active, double* relres, int* iters, int* conv,
                      double* hist, int it, double tol, int* ctl, int k, cudaStream_t s);
void launch_pcg_beta(const double* rzn, double* rz, const int* active, double* beta, int* ctl, int it, int k,
                     cudaStream_t s);
void launch_ratio(const double* num, const double* den, const int* active, double* out, int k, cudaStream_t s);
void launch_xmy(double* y, const double* x, int64_t n, cudaStream_t s);
void launch_scale(double* y, const double* x, const double* nrm2, int64_t n, cudaStream_t s);

}  // namespace phif
