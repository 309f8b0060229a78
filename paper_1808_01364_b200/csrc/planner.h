// Host-side level planner for the B200 PHIF engine (pure C++, no CUDA).
//
// Restates the reference grouping (hierarchy.py:102-168) and derives, per
// level, everything the batched stage kernels need: groups in classify order
// with ascending members, the symbolic block pattern of the live matrix
// (dense blocks keyed (g,h), g <= h), cell/boundary lists,
// Schur-target contribution lists, skeleton neighbour lists and the
// dependency wavefronts of the sequential skeletonization.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace phif {

struct Spec {
  int dim = 2, n = 0, m = 0, L = 0;
  int64_t N = 0;  // (n-1)^dim
  void init(int d, int nn, int mm);
};

// kind = number of on-line axes: 0 interior, 1 edge(2D)/face(3D), 2 corner(2D)/edge(3D), 3 corner(3D)
struct Groups {
  int level = 0;
  int G = 0;
  std::vector<int> q;      // 3*G cell coordinates
  std::vector<int> bits;   // on-line mask
  std::vector<int> kind;
  std::vector<int64_t> off;   // G+1
  std::vector<int> mem;       // members, ascending within a group
  // level transition provenance (empty at level 0): per member, source group in the
  // previous level and the member's position inside that source's full member list
  std::vector<int> src_group;
  std::vector<int> src_pos;
  std::vector<int> src_local;      // index of src_group in the new group's source list
  std::vector<int64_t> srcl_off;    // G+1: distinct source groups of each new group
  std::vector<int> srcl;
  int size(int g) const { return (int)(off[g + 1] - off[g]); }
  bool is_sep(int g, int dim) const { return kind[g] == 1; }
};

struct Pattern {
  std::vector<int> bg, bh;          // block (bg[b], bh[b]) with bg <= bh, sorted
  std::vector<int64_t> adj_off;     // per group CSR (G+1)
  std::vector<int> adj_nbr, adj_blk; // neighbour group and block id, sorted by neighbour
  int find(int g, int h) const;     // block id of (min,max) or -1
};

struct LevelPlan {
  int level = 0;
  bool root = false;
  Groups grp;
  Pattern pat;             // all blocks at this level (input pattern + elimination fill)
  std::vector<int64_t> boff;  // pool offset (doubles) per block
  int64_t pool_doubles = 0;
  std::vector<int> interior, precond, skeleton;  // group ids, classify order
  // cells (stage 1): per interior t: neighbour groups (ascending) -> B
  std::vector<int64_t> cell_nbr_off;  // p+1
  std::vector<int> cell_nbr;          // neighbour group ids
  std::vector<int> cell_nbr_blk;      // block (I, h)
  std::vector<int> cell_nbr_col;      // column offset of h inside B
  std::vector<int> cell_n, cell_b;
  // Schur assembly: per target block, contributions (cell t, row off, col off) in cell order
  std::vector<int> tgt_blk;
  std::vector<int64_t> tgt_off;       // per target (size ntargets+1)
  std::vector<int> con_cell, con_row, con_col;
  std::vector<int> con_ri, con_ci;    // (host only) neighbour index of the row / column group in its cell
  // off-diagonal blocks scaled by block Jacobi (both ends preconditioned)
  std::vector<int> scale_blk;
  // skeletonization: per skeleton s: neighbour (h, blk) lists excluding self, wave index
  std::vector<int64_t> sk_nbr_off;
  std::vector<int> sk_nbr, sk_nbr_blk;
  std::vector<int> sk_wave;
  int nwaves = 0;
  std::vector<int> wave_order;        // skeleton indices sorted by (wave, index)
  std::vector<int64_t> wave_off;      // nwaves+1 into wave_order
  // dependency graph of the sequential skeletonization: earlier coupled separators (count) and
  // later coupled separators (lists), for dependency-driven scheduling
  std::vector<int> sk_ndep;
  std::vector<int64_t> sk_succ_off;
  std::vector<int> sk_succ;
};

// level 0 grouping of all DOFs
Groups classify_all(const Spec& s);
// grouping of an arbitrary active set at `level` (hierarchy.py:102 semantics)
Groups classify_set(const Spec& s, int level, const std::vector<int>& active);
// next level grouping from survivors; alive[pos] over grp.mem (1 = survives)
Groups classify_next(const Spec& s, const Groups& prev, const std::vector<uint8_t>& alive);
// block pattern at level 0 from the CSR pattern of A
std::vector<std::pair<int, int>> pattern_from_csr(const Groups& g, int64_t N, const int64_t* rowptr,
                                                  const int* col);
// map the surviving pattern of the previous level onto the next grouping
std::vector<std::pair<int, int>> pattern_next(const LevelPlan& prev, const Groups& next);
// complete a level plan from its groups and input pattern
void build_level(const Spec& s, LevelPlan& lp, std::vector<std::pair<int, int>> pairs);

// Pre-plan of level l+1 computed while level l's IDs run: the grouping and every structural list
// of the next level assuming each non-interior group of level l keeps all its DOFs (group pairs,
// adjacency, cells, Schur targets, scaling blocks, skeleton lists and wavefronts depend only on
// which groups exist, not on their sizes).
LevelPlan preplan_next(const Spec& s, const LevelPlan& prev);
// Finish a pre-plan with the real survivors: drop the redundant members (ascending order and
// provenance kept) and recompute what depends on group sizes (pool offsets, cell sizes and
// boundary columns, Schur contribution columns). Returns false if some non-interior group of the
// previous level lost every DOF (the grouping changes; re-plan from scratch).
bool finish_preplan(const Spec& s, LevelPlan& lp, const LevelPlan& prev, const std::vector<uint8_t>& alive);

std::string level_json(const LevelPlan& lp);

// dependency wavefronts of the sequential skeletonization (sk_wave, nwaves, wave_off, wave_order)
// from the skeleton neighbour lists (build_level does this itself; the device planner leaves it)
void compute_waves(LevelPlan& lp, int G);

// Host vector pool for plan arrays: vectors taken from it are reused allocations (already
// faulted in), so large per-factorization plan arrays cost a copy, not fresh page faults.
// pool_take returns a vector of size n with unspecified contents; recycle_plan gives every
// array of a finished plan back.
std::vector<int> pool_take_int(size_t n);
std::vector<int64_t> pool_take_i64(size_t n);
void recycle_plan(LevelPlan& lp);

}  // namespace phif
