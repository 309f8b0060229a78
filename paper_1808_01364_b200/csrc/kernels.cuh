// Kernel parameter blocks and launch wrappers of the B200 PHIF engine.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace phif {

// Status word: (op << 32 | pivot) of the lowest failing op; ~0ull when none.
struct DevStatus {
  unsigned long long first_bad;
};

struct LevelDev {
  // groups
  int G;
  const int64_t* goff;   // G+1
  const int* mem;        // members
  const int* gsize;      // G
  // blocks
  double* pool;
  const int64_t* boff;
  const int* bg;
  const int* bh;
  const int64_t* adj_off;
  const int* adj_nbr;
  const int* adj_blk;
  const int* diag_blk;   // per group: block id of (g,g)
};

struct CellArgs {
  int p;
  const int* list;          // cells handled by the one-CTA kernel (nullptr = all)
  const int* interior;      // group ids
  const int64_t* nbr_off;   // p+1
  const int* nbr_blk;
  const int* nbr_col;
  const int* nbr_w;
  const int* n;
  const int* b;
  double* rec;              // record pool
  const int64_t* P_off;     // panel (n+b) x n
  double* U;                // Schur workspace
  const int64_t* U_off;     // b x b
};

struct SchurArgs {
  int ntgt;
  const int* tgt_blk;
  const int64_t* tgt_off;
  const int* con_cell;
  const int* con_row;
  const int* con_col;
  const int* cell_b;
  const double* U;
  const int64_t* U_off;
};

struct PrecArgs {
  int r;
  const int* list;                // groups factored by the one-CTA kernel (nullptr = all)
  const int* scale_list;          // blocks scaled by the one-CTA kernel (nullptr = all)
  const int* groups;
  double* rec;
  const int64_t* L_off;           // per precond index
  const int64_t* L_off_of_group;  // per group id (-1 if none)
  int nscale;
  const int* scale_blk;
};

struct SkelArgs {
  int nsk;
  const int* groups;         // skeleton group ids
  const int64_t* nbr_off;
  const int* nbr;
  const int* nbr_blk;
  const int* order;          // wave order slice
  int* alive;                // per DOF (global)
  uint8_t* red;              // per member position of the level (1 = redundant)
  int* rank;                 // per skeleton
  int* rows;                 // per skeleton: rows of A_{R,I} after filtering
  double eps;
  int gram;                  // 1: separators of <= 57 columns take the Gram-path ID (skel_id_gram)
  long long* prof;           // optional phase clocks (PHIF_GID_PROF), slots 16..23
  double* work;              // per skeleton workspace
  const int64_t* work_off;
  int* iwork;
  const int64_t* iwork_off;
  double* rec;
  const int64_t* T_off;      // r x kt
  const int64_t* P_off;      // (kt + r) x kt
};

// dependency-driven scheduling of separator IDs (k_skel_id_dyn)
struct DynSched {
  int count;             // separators (sk.order[0..count) in topological order)
  int* next;             // work counter (zeroed)
  int* done;             // per separator: finished earlier coupled separators (zeroed)
  const int* ndep;       // per separator: earlier coupled separators
  const int64_t* succ_off;
  const int* succ;       // later coupled separators
};

struct TeamHdr {
  unsigned count;
  unsigned gen;
  unsigned qr_done;   // panels of the row-reduction QR published so far
  double tau;
};

struct TeamArgs {
  int nface;
  const int* face;       // skeleton index per team
  const int* team_off;   // nface+1 CTA offsets
  TeamHdr* hdr;          // per team
  double* slot_v;        // 2 per CTA (double-buffered by step parity)
  int* slot_i;           // 2 per CTA
  int vcap;              // Householder vector staged in smem when m <= vcap
  int kmax;              // largest separator of the launch (replicated permutation in smem)
  long long* prof;       // optional per-phase clock accumulators (debug)
  double* cand;          // 2 staging columns per CTA (pivot candidates), ld cand_ld
  int64_t cand_ld;
  int colcap;            // doubles of shared memory for resident owned columns
  double* qt;            // per team: T factors of the QR panels, qt_ld doubles
  int64_t qt_ld;
  int cluster;           // > 0: teams are thread-block clusters of this size (cluster barriers)
};

// Gram-path ID of large separators (gram_id.cuh): one wave's items
struct GramArgs {
  int nitem;
  const int* item_sep;     // skeleton index per item
  const int64_t* item_ld;  // leading dimension of the gathered A_{R,I} (rows bound)
  int P;                   // gather CTAs per item
  int* cnt;                // nitem * P kept-row counts
  double* gbuf;            // per item: G (k x k, then R) [+ packed Schur complement when global]
  const int64_t* g_off;
  const int* w_item;       // Gram tile work list (lower 64x64 tiles)
  const int* w_i;
  const int* w_j;
  int nwork;
  int C;                   // CPQR cluster size
  int S;                   // split-K factor of the Gram tiles (partial G blocks summed by the CPQR)
  int nb;                  // deferred-update panel width (<= 16)
  int* col;                // per item: column at every pivot position (read by k_gid_T)
  const int64_t* c_off;
  int CT;                  // k_gid_T: CTAs per item
  int64_t tcap;            // k_gid_T: staging doubles per CTA
  long long* prof;         // optional phase clocks of CTA 0 (PHIF_GID_PROF)
};

struct RepackArgs {
  int nblk;
  // work items: row chunks of new blocks
  int nwork;
  const int* w_blk;
  const int* w_row0;
  const int* w_nrow;
  int tab_cap;                  // max (#source groups of G) x (#source groups of H)
  const int* nsrc_local;        // per new member: index into its group's source list
  const int64_t* nsrcl_off;     // per new group: range of distinct source groups
  const int* nsrcl;
  // new level
  const int* nbg;
  const int* nbh;
  const int64_t* nboff;
  const int64_t* ngoff;
  const int* nsrc_group;   // per new member
  const int* nsrc_pos;
  double* npool;
  // old level
  const double* opool;
  const int64_t* oboff;
  const int64_t* oadj_off;
  const int* oadj_nbr;
  const int* oadj_blk;
  const int* ogsize;
};

}  // namespace phif

namespace phif {

// Tile-parallel path for big cells (one level's big cells batched): the panel
// P_c ((n+b) x n row-major, ld n) is factored right-looking in 64-wide steps.
struct BigArgs {
  int ncell;
  const int* n;            // per big cell
  const int* b;
  const int* rows;         // panel rows: n + b (+ n identity rows whose result is L^-T)
  double* const* P;        // panel base per big cell
  double* const* U;        // Schur output per big cell (b x b)
  double* Linv;            // 64 x 64 scratch per big cell
  const int* op;           // original op index (status reporting)
  // per-step tile work list: (cell, row tile, col tile)
  const int* w_cell;
  const int* w_i;
  const int* w_j;
  int nwork;
  int k0;                  // current step's panel start
  int kw;                  // update depth (columns k0 .. k0+kw)
};

}  // namespace phif

namespace phif {

// Generic batched GEMM work: C = beta*C + alpha*op(A)*B, tile-parallel over 64-row tiles.
struct GemmDesc {
  const double* A;
  const double* B;
  double* C;
  int M, N, K, lda, ldb, ldc;
  int transA;
  double alpha, beta;
  int tri = 0;   // 0 dense; 1: op(A) lower (K < tile's last row); 2: B upper (K < tile's last column);
                 // 3: op(A) upper (K >= tile's first row)
};

}  // namespace phif
