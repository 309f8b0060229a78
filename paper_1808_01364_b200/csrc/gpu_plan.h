// Device-side level-0 planner (gpu_plan.cu): the level-0 LevelPlan computed on the GPU.
#pragma once
#include "engine.h"
#include "planner.h"

namespace phif {

// Level-0 plan arrays resident in HBM (moved into the LevelRT buffers by factorize()).
struct DevPlan0 {
  bool valid = false;
  DBuf goff, mem, gsize, kind;
  DBuf bg, bh, boff, adj_off, adj_nbr, adj_blk, diag_blk;
  DBuf interior, precond, skeleton;
  DBuf cell_nbr_off, cell_nbr, cell_nbr_blk, cell_nbr_col, cell_nbr_w, cell_n, cell_b;
  DBuf tgt_blk, tgt_off, con_cell, con_row, con_col;
  DBuf scale_blk;
  DBuf sk_nbr_off, sk_nbr, sk_nbr_blk, sk_ndep, sk_succ_off, sk_succ;
  int64_t nblocks = 0, ncon = 0, nsk_nbr = 0, nsucc = 0;
  int ntgt = 0, nscale = 0;
};

// the device planner handles level 0 when its cells take the one-CTA path
bool gpu_plan0_applicable(const Spec& s, int big_cell);

// Plan level 0 on the device from the device CSR pattern. Fills `dp` and the host fields of `lp`
// the level loop reads (groups, block pairs, interior/precond/skeleton lists, cell lists, Schur
// target blocks, scaling blocks, skeleton neighbour lists, dependency wavefronts); the adjacency,
// pool offsets, cell block/column lists, Schur contribution lists and dependency lists stay on
// the device only.
void plan_level0_device(const Spec& s, const int64_t* rowptr, const int* col, int64_t nnz, LevelPlan& lp,
                        DevPlan0& dp, cudaStream_t st);

// Copy the device-only arrays of `dp` into `lp` too (planner check).
void download_plan0(DevPlan0& dp, LevelPlan& lp, cudaStream_t st);

}  // namespace phif
