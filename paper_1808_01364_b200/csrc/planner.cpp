#include <chrono>
#include <cstdio>
#include <cstdlib>
// Host-side level planner (see planner.h).
#include "planner.h"

#include <algorithm>
#include <cstdio>
#include <numeric>
#include <sstream>
#include <stdexcept>
#include <tuple>

namespace phif {

void Spec::init(int d, int nn, int mm) {
  dim = d;
  n = nn;
  m = mm;
  int cells = n / m, l = 0;
  while ((1 << (l + 1)) <= cells) ++l;
  L = l;
  N = 1;
  for (int i = 0; i < dim; ++i) N *= (n - 1);
}

namespace {

struct KeyInfo {
  int per, sz;
};

inline void coords_of(const Spec& s, int64_t dof, int c[3]) {
  const int64_t side = s.n - 1;
  c[0] = (int)(dof % side) + 1;
  c[1] = (int)((dof / side) % side) + 1;
  c[2] = s.dim == 3 ? (int)(dof / (side * side)) + 1 : 0;
}

// group key (x-major cell index, kind bits last), hierarchy.py:124-133
inline int64_t key_of(const Spec& s, int level, int64_t dof, int q[3], int& bits) {
  const int sz = s.m << level, per = s.n / sz;
  int c[3];
  coords_of(s, dof, c);
  bits = 0;
  int64_t key = 0;
  for (int d = 0; d < s.dim; ++d) {
    q[d] = c[d] / sz;
    if (c[d] % sz == 0) bits |= 1 << d;
    key = key * per + q[d];
  }
  return (key << s.dim) | bits;
}

inline int popc(int b) { return __builtin_popcount((unsigned)b); }

void finalize_groups(const Spec& s, Groups& g, const std::vector<int64_t>& keys_sorted_members,
                     const std::vector<int64_t>& key_of_group) {
  (void)keys_sorted_members;
  g.G = (int)key_of_group.size();
  g.q.assign(3 * (size_t)g.G, 0);
  g.bits.assign(g.G, 0);
  g.kind.assign(g.G, 0);
  for (int i = 0; i < g.G; ++i) {
    int q[3] = {0, 0, 0}, b = 0;
    key_of(s, g.level, g.mem[g.off[i]], q, b);
    for (int d = 0; d < 3; ++d) g.q[3 * i + d] = q[d];
    g.bits[i] = b;
    g.kind[i] = popc(b);
  }
}

}  // namespace

Groups classify_all(const Spec& s) {
  Groups g;
  g.level = 0;
  const int sz = s.m, per = s.n / sz;
  int64_t nkeys = 1;
  for (int d = 0; d < s.dim; ++d) nkeys *= per;
  nkeys <<= s.dim;
  std::vector<int> key(s.N);
  std::vector<int64_t> cnt(nkeys + 1, 0);
  {
    // per-axis tables: cell index and on-line bit of every lattice coordinate
    const int side = s.n - 1;
    std::vector<int> qa(side + 1), ba(side + 1);
    for (int c = 1; c <= side; ++c) {
      qa[c] = c / sz;
      ba[c] = (c % sz == 0) ? 1 : 0;
    }
    const int64_t plane = (int64_t)side * side;
    const int nz = s.dim == 3 ? side : 1;
#pragma omp parallel for schedule(static)
    for (int64_t yz = 0; yz < (int64_t)side * nz; ++yz) {
      const int y = (int)(yz % side) + 1, z = s.dim == 3 ? (int)(yz / side) + 1 : 0;
      int64_t base = 0;
      int bits_yz = 0;
      if (s.dim == 2) {
        base = 0;
        bits_yz = ba[y] << 1;
      } else {
        base = 0;
        bits_yz = (ba[y] << 1) | (ba[z] << 2);
      }
      const int64_t row0 = (int64_t)(y - 1) * side + (s.dim == 3 ? (int64_t)(z - 1) * plane : 0);
      for (int x = 1; x <= side; ++x) {
        int64_t k = qa[x];
        k = k * per + qa[y];
        if (s.dim == 3) k = k * per + qa[z];
        key[row0 + x - 1] = (int)((k << s.dim) | (ba[x] | bits_yz));
      }
      (void)base;
    }
    for (int64_t i = 0; i < s.N; ++i) cnt[key[i] + 1]++;
  }
  for (int64_t k = 0; k < nkeys; ++k) cnt[k + 1] += cnt[k];
  g.mem.resize(s.N);
  std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
  for (int64_t i = 0; i < s.N; ++i) g.mem[fill[key[i]]++] = (int)i;
  std::vector<int64_t> gkeys;
  g.off.clear();
  for (int64_t k = 0; k < nkeys; ++k)
    if (cnt[k + 1] > cnt[k]) {
      gkeys.push_back(k);
      g.off.push_back(cnt[k]);
    }
  g.off.push_back(s.N);
  finalize_groups(s, g, {}, gkeys);
  return g;
}

Groups classify_set(const Spec& s, int level, const std::vector<int>& active) {
  Groups g;
  g.level = level;
  std::vector<std::pair<int64_t, int>> items;
  items.reserve(active.size());
  for (int dof : active) {
    if (dof < 0 || dof >= s.N) throw std::runtime_error("classify: DOF outside the domain");
    int q[3], b;
    items.emplace_back(key_of(s, level, dof, q, b), dof);
  }
  std::sort(items.begin(), items.end());
  std::vector<int64_t> gkeys;
  g.mem.resize(items.size());
  for (size_t i = 0; i < items.size(); ++i) {
    if (i == 0 || items[i].first != items[i - 1].first) {
      gkeys.push_back(items[i].first);
      g.off.push_back((int64_t)i);
    }
    g.mem[i] = items[i].second;
  }
  g.off.push_back((int64_t)items.size());
  finalize_groups(s, g, {}, gkeys);
  return g;
}

Groups classify_next(const Spec& s, const Groups& prev, const std::vector<uint8_t>& alive) {
  // Every surviving DOF of an old group lands in the same new group (the old group's
  // on-line axes stay on-line iff their line index is even; free coordinates stay inside
  // the same cell), so the new grouping is a bucket sort of old groups by their new key
  // followed by a per-group merge of survivors in ascending DOF order (hierarchy.py:145).
  Groups g;
  g.level = prev.level + 1;
  const int per = s.n / (s.m << g.level);
  int64_t nkeys = 1;
  for (int d = 0; d < s.dim; ++d) nkeys *= per;
  nkeys <<= s.dim;
  std::vector<int64_t> okey(prev.G, -1);
  std::vector<int> osurv(prev.G, 0);
#pragma omp parallel for schedule(static)
  for (int pg = 0; pg < prev.G; ++pg) {
    int cnt = 0;
    int64_t first = -1;
    for (int64_t p = prev.off[pg]; p < prev.off[pg + 1]; ++p)
      if (alive[p]) {
        if (cnt == 0) first = p;
        ++cnt;
      }
    osurv[pg] = cnt;
    if (cnt) {
      int q[3], b;
      okey[pg] = key_of(s, g.level, prev.mem[first], q, b);
    }
  }
  // bucket old groups by new key (stable: ascending old group index)
  std::vector<int64_t> kcnt(nkeys + 1, 0);
  for (int pg = 0; pg < prev.G; ++pg)
    if (okey[pg] >= 0) kcnt[okey[pg] + 1]++;
  for (int64_t k = 0; k < nkeys; ++k) kcnt[k + 1] += kcnt[k];
  std::vector<int> order(kcnt[nkeys]);
  {
    std::vector<int64_t> fill(kcnt.begin(), kcnt.end() - 1);
    for (int pg = 0; pg < prev.G; ++pg)
      if (okey[pg] >= 0) order[fill[okey[pg]]++] = pg;
  }
  std::vector<int64_t> gkeys;
  std::vector<int64_t> gsrc_off;   // new group -> range in `order`
  int64_t total = 0;
  std::vector<int64_t> moff;
  for (int64_t k = 0; k < nkeys; ++k)
    if (kcnt[k + 1] > kcnt[k]) {
      gkeys.push_back(k);
      gsrc_off.push_back(kcnt[k]);
      moff.push_back(total);
      for (int64_t q = kcnt[k]; q < kcnt[k + 1]; ++q) total += osurv[order[q]];
    }
  gsrc_off.push_back(kcnt[nkeys]);
  moff.push_back(total);
  const int G = (int)gkeys.size();
  g.off = moff;
  g.mem.resize(total);
  g.src_group.resize(total);
  g.src_pos.resize(total);
  g.src_local.resize(total);
  g.srcl_off.assign(gsrc_off.begin(), gsrc_off.end());
  g.srcl.assign(order.begin(), order.end());
#pragma omp parallel
  {
    std::vector<std::tuple<int, int, int>> seg;
#pragma omp for schedule(dynamic, 64)
    for (int G0 = 0; G0 < G; ++G0) {
      seg.clear();
      for (int64_t q = gsrc_off[G0]; q < gsrc_off[G0 + 1]; ++q) {
        const int pg = order[q];
        for (int64_t p = prev.off[pg]; p < prev.off[pg + 1]; ++p)
          if (alive[p]) seg.emplace_back(prev.mem[p], (int)(q - gsrc_off[G0]), (int)(p - prev.off[pg]));
      }
      std::sort(seg.begin(), seg.end());
      int64_t o = g.off[G0];
      for (auto& t : seg) {
        g.mem[o] = std::get<0>(t);
        g.src_local[o] = std::get<1>(t);
        g.src_group[o] = order[gsrc_off[G0] + std::get<1>(t)];
        g.src_pos[o] = std::get<2>(t);
        ++o;
      }
    }
  }
  finalize_groups(s, g, {}, gkeys);
  return g;
}

int Pattern::find(int g, int h) const {
  if (g > h) std::swap(g, h);
  const int* b = adj_nbr.data() + adj_off[g];
  const int* e = adj_nbr.data() + adj_off[g + 1];
  const int* it = std::lower_bound(b, e, h);
  if (it == e || *it != h) return -1;
  return adj_blk[adj_off[g] + (it - adj_nbr.data() - adj_off[g])];
}

std::vector<std::pair<int, int>> pattern_from_csr(const Groups& g, int64_t N, const int64_t* rowptr,
                                                  const int* col) {
  std::vector<int> gid(N, -1);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < g.G; ++i)
    for (int64_t p = g.off[i]; p < g.off[i + 1]; ++p) gid[g.mem[p]] = i;
  std::vector<std::pair<int, int>> pairs;
#pragma omp parallel
  {
    std::vector<std::pair<int, int>> mine;
    std::vector<int> seen;
#pragma omp for schedule(static) nowait
    for (int i = 0; i < g.G; ++i) {
      seen.clear();
      for (int64_t p = g.off[i]; p < g.off[i + 1]; ++p) {
        const int r = g.mem[p];
        for (int64_t e = rowptr[r]; e < rowptr[r + 1]; ++e) {
          const int h = gid[col[e]];
          if (h >= i && std::find(seen.begin(), seen.end(), h) == seen.end()) seen.push_back(h);
        }
      }
      for (int h : seen) mine.emplace_back(i, h);
    }
#pragma omp critical
    pairs.insert(pairs.end(), mine.begin(), mine.end());
  }
  return pairs;
}

std::vector<std::pair<int, int>> pattern_next(const LevelPlan& prev, const Groups& next) {
  std::vector<int> old2new(prev.grp.G, -1);
  for (int G = 0; G < next.G; ++G)
    for (int64_t p = next.off[G]; p < next.off[G + 1]; ++p) {
      const int og = next.src_group[p];
      if (old2new[og] >= 0 && old2new[og] != G)
        throw std::runtime_error("planner: an old group split across new groups");
      old2new[og] = G;
    }
  std::vector<std::pair<int, int>> pairs;
  pairs.reserve(prev.pat.bg.size());
  for (size_t b = 0; b < prev.pat.bg.size(); ++b) {
    const int og = prev.pat.bg[b], oh = prev.pat.bh[b];
    if (prev.grp.kind[og] == 0 || prev.grp.kind[oh] == 0) continue;
    const int G = old2new[og], H = old2new[oh];
    if (G < 0 || H < 0) continue;
    pairs.emplace_back(std::min(G, H), std::max(G, H));
  }
  return pairs;
}

static void sort_unique(std::vector<std::pair<int, int>>& v) {
  std::sort(v.begin(), v.end());
  v.erase(std::unique(v.begin(), v.end()), v.end());
}

static void build_adjacency(int G, const std::vector<std::pair<int, int>>& pairs, Pattern& pat) {
  pat.bg.resize(pairs.size());
  pat.bh.resize(pairs.size());
  std::vector<int64_t> deg(G + 1, 0);
  for (size_t b = 0; b < pairs.size(); ++b) {
    pat.bg[b] = pairs[b].first;
    pat.bh[b] = pairs[b].second;
    deg[pairs[b].first + 1]++;
    if (pairs[b].first != pairs[b].second) deg[pairs[b].second + 1]++;
  }
  for (int i = 0; i < G; ++i) deg[i + 1] += deg[i];
  pat.adj_off = deg;
  pat.adj_nbr.assign(deg[G], 0);
  pat.adj_blk.assign(deg[G], 0);
  std::vector<int64_t> fill(deg.begin(), deg.end() - 1);
  // pairs are sorted by (g,h): for each g, entries (g,h) arrive in ascending h, but the
  // reverse entries (h -> g) interleave, so sort each row afterwards
  for (size_t b = 0; b < pairs.size(); ++b) {
    const int g = pairs[b].first, h = pairs[b].second;
    pat.adj_nbr[fill[g]] = h;
    pat.adj_blk[fill[g]++] = (int)b;
    if (g != h) {
      pat.adj_nbr[fill[h]] = g;
      pat.adj_blk[fill[h]++] = (int)b;
    }
  }
  std::vector<std::pair<int, int>> tmp;
  for (int g = 0; g < G; ++g) {
    const int64_t a = deg[g], e = deg[g + 1];
    tmp.clear();
    for (int64_t p = a; p < e; ++p) tmp.emplace_back(pat.adj_nbr[p], pat.adj_blk[p]);
    std::sort(tmp.begin(), tmp.end());
    for (int64_t p = a; p < e; ++p) {
      pat.adj_nbr[p] = tmp[p - a].first;
      pat.adj_blk[p] = tmp[p - a].second;
    }
  }
}

// per-group sorted, de-duplicated "upper" neighbour lists (h >= g) from unsorted pairs
static void upper_lists(int G, const std::vector<std::pair<int, int>>& pairs, std::vector<int64_t>& off,
                        std::vector<int>& nbr) {
  off.assign(G + 1, 0);
  for (const auto& pr : pairs) off[pr.first + 1]++;
  for (int i = 0; i < G; ++i) off[i + 1] += off[i];
  nbr.assign(off[G], 0);
  {
    std::vector<int64_t> fill(off.begin(), off.end() - 1);
    for (const auto& pr : pairs) nbr[fill[pr.first]++] = pr.second;
  }
  std::vector<int64_t> keep(G + 1, 0);
#pragma omp parallel for schedule(dynamic, 256)
  for (int gi = 0; gi < G; ++gi) {
    int* b = nbr.data() + off[gi];
    int* e = nbr.data() + off[gi + 1];
    std::sort(b, e);
    keep[gi + 1] = std::unique(b, e) - b;
  }
  for (int i = 0; i < G; ++i) keep[i + 1] += keep[i];
  std::vector<int> out(keep[G]);
#pragma omp parallel for schedule(static)
  for (int gi = 0; gi < G; ++gi)
    std::copy(nbr.begin() + off[gi], nbr.begin() + off[gi] + (keep[gi + 1] - keep[gi]), out.begin() + keep[gi]);
  off.swap(keep);
  nbr.swap(out);
}

// symmetric adjacency (rows sorted by neighbour) from upper lists; block ids in (g, h) order
static void adjacency_from_upper(int G, const std::vector<int64_t>& uoff, const std::vector<int>& unbr,
                                 Pattern& pat) {
  const int64_t nb = uoff[G];
  pat.bg.resize(nb);
  pat.bh.resize(nb);
  std::vector<int64_t> ndown(G + 1, 0);
  for (int gi = 0; gi < G; ++gi)
    for (int64_t q = uoff[gi]; q < uoff[gi + 1]; ++q) {
      pat.bg[q] = gi;
      pat.bh[q] = unbr[q];
      if (unbr[q] != gi) ndown[unbr[q] + 1]++;
    }
  pat.adj_off.assign(G + 1, 0);
  for (int gi = 0; gi < G; ++gi) pat.adj_off[gi + 1] = pat.adj_off[gi] + ndown[gi + 1] + (uoff[gi + 1] - uoff[gi]);
  pat.adj_nbr.assign(pat.adj_off[G], 0);
  pat.adj_blk.assign(pat.adj_off[G], 0);
  std::vector<int64_t> fill(pat.adj_off.begin(), pat.adj_off.end() - 1);
  // lower neighbours first, in increasing order (outer loop over ascending g)
  for (int gi = 0; gi < G; ++gi)
    for (int64_t q = uoff[gi]; q < uoff[gi + 1]; ++q) {
      const int h = unbr[q];
      if (h == gi) continue;
      pat.adj_nbr[fill[h]] = gi;
      pat.adj_blk[fill[h]++] = (int)q;
    }
#pragma omp parallel for schedule(static)
  for (int gi = 0; gi < G; ++gi) {
    int64_t f = fill[gi];
    for (int64_t q = uoff[gi]; q < uoff[gi + 1]; ++q) {
      pat.adj_nbr[f] = unbr[q];
      pat.adj_blk[f++] = (int)q;
    }
  }
}

void build_level(const Spec& s, LevelPlan& lp, std::vector<std::pair<int, int>> pairs) {
  const bool tdbg = getenv("PHIF_PLAN_TIMING") != nullptr;
  auto tl = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!tdbg) return;
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "  [plan L%d] %-28s %8.2f ms\n", lp.grp.level, what, std::chrono::duration<double, std::milli>(now - tl).count());
    tl = now;
  };
  Groups& g = lp.grp;
  lp.level = g.level;
  lp.root = (g.level == s.L);
  for (int i = 0; i < g.G; ++i) pairs.emplace_back(i, i);
  std::vector<int64_t> uoff;
  std::vector<int> unbr;
  lap("upper lists (stencil)");
  upper_lists(g.G, pairs, uoff, unbr);
  lp.interior.clear();
  lp.precond.clear();
  lp.skeleton.clear();
  for (int i = 0; i < g.G; ++i) {
    if (g.kind[i] == 0) {
      lp.interior.push_back(i);
    } else {
      lp.precond.push_back(i);
      if (g.kind[i] == 1) lp.skeleton.push_back(i);
    }
  }
  // an interior group is the first group of its cell closure: every coupling of it is an upper entry
  for (int gi = 0; gi < g.G; ++gi)
    for (int64_t q = uoff[gi]; q < uoff[gi + 1]; ++q)
      if (unbr[q] != gi && g.kind[unbr[q]] == 0)
        throw std::runtime_error(g.kind[gi] == 0 ? "planner: two interior groups coupled"
                                                 : "planner: interior group is not first in its closure");
  lap("classify + checks");
  // elimination fill among each cell's boundary groups
  pairs.clear();
  for (int gi = 0; gi < g.G; ++gi)
    for (int64_t q = uoff[gi]; q < uoff[gi + 1]; ++q) pairs.emplace_back(gi, unbr[q]);
  for (int I : lp.interior) {
    const int64_t a0 = uoff[I], a1 = uoff[I + 1];
    for (int64_t a = a0; a < a1; ++a) {
      if (unbr[a] == I) continue;
      for (int64_t b = a; b < a1; ++b) pairs.emplace_back(unbr[a], unbr[b]);
    }
  }
  lap("fill pairs");
  upper_lists(g.G, pairs, uoff, unbr);
  adjacency_from_upper(g.G, uoff, unbr, lp.pat);
  lap("adjacency");
  const Pattern& pat = lp.pat;
  const int64_t nblocks = (int64_t)pat.bg.size();
  // pool
  lp.boff.resize(nblocks);
  int64_t acc = 0;
  for (int64_t b = 0; b < nblocks; ++b) {
    lp.boff[b] = acc;
    acc += (int64_t)g.size(pat.bg[b]) * g.size(pat.bh[b]);
  }
  lp.pool_doubles = acc;
  lap("pool");
  // cells: boundary = neighbour groups of I (all after I); Schur targets = pairs of them
  const int p = (int)lp.interior.size();
  lp.cell_nbr_off.assign(p + 1, 0);
  lp.cell_n.assign(p, 0);
  lp.cell_b.assign(p, 0);
  for (int t = 0; t < p; ++t) {
    const int I = lp.interior[t];
    lp.cell_nbr_off[t + 1] = lp.cell_nbr_off[t] + (uoff[I + 1] - uoff[I] - 1);
  }
  const int64_t ncn = lp.cell_nbr_off[p];
  lp.cell_nbr.assign(ncn, 0);
  lp.cell_nbr_blk.assign(ncn, 0);
  lp.cell_nbr_col.assign(ncn, 0);
  std::vector<int64_t> ccount(p + 1, 0);
#pragma omp parallel for schedule(static)
  for (int t = 0; t < p; ++t) {
    const int I = lp.interior[t];
    int64_t o = lp.cell_nbr_off[t];
    int bcols = 0;
    for (int64_t q = uoff[I]; q < uoff[I + 1]; ++q) {
      const int h = unbr[q];
      if (h == I) continue;
      lp.cell_nbr[o] = h;
      lp.cell_nbr_blk[o] = (int)q;
      lp.cell_nbr_col[o] = bcols;
      bcols += g.size(h);
      ++o;
    }
    lp.cell_n[t] = g.size(I);
    lp.cell_b[t] = bcols;
    const int64_t w = lp.cell_nbr_off[t + 1] - lp.cell_nbr_off[t];
    ccount[t + 1] = w * (w + 1) / 2;
  }
  for (int t = 0; t < p; ++t) ccount[t + 1] += ccount[t];
  const int64_t ncons = ccount[p];
  std::vector<int> ctgt(ncons), ccell(ncons), crow(ncons), ccol(ncons);
#pragma omp parallel for schedule(static)
  for (int t = 0; t < p; ++t) {
    int64_t o = ccount[t];
    const int64_t first = lp.cell_nbr_off[t], last = lp.cell_nbr_off[t + 1];
    for (int64_t a = first; a < last; ++a) {
      const int ha = lp.cell_nbr[a];
      const int* rb = unbr.data() + uoff[ha];
      const int* re = unbr.data() + uoff[ha + 1];
      for (int64_t b = a; b < last; ++b) {
        const int* it = std::lower_bound(rb, re, lp.cell_nbr[b]);
        ctgt[o] = (int)(it - unbr.data());   // block id = position in the upper lists
        ccell[o] = t;
        crow[o] = lp.cell_nbr_col[a];
        ccol[o] = lp.cell_nbr_col[b];
        ++o;
      }
    }
  }
  lap("cells + contributions");
  // group contributions by target block (counting sort; stable in cell order)
  std::vector<int64_t> tcnt(nblocks + 1, 0);
  for (int64_t i = 0; i < ncons; ++i) tcnt[ctgt[i] + 1]++;
  for (int64_t b = 0; b < nblocks; ++b) tcnt[b + 1] += tcnt[b];
  lp.con_cell.resize(ncons);
  lp.con_row.resize(ncons);
  lp.con_col.resize(ncons);
  {
    std::vector<int64_t> fill(tcnt.begin(), tcnt.end() - 1);
    for (int64_t i = 0; i < ncons; ++i) {
      const int64_t o = fill[ctgt[i]]++;
      lp.con_cell[o] = ccell[i];
      lp.con_row[o] = crow[i];
      lp.con_col[o] = ccol[i];
    }
  }
  lp.tgt_blk.clear();
  lp.tgt_off.assign(1, 0);
  for (int64_t b = 0; b < nblocks; ++b)
    if (tcnt[b + 1] > tcnt[b]) {
      lp.tgt_blk.push_back((int)b);
      lp.tgt_off.push_back(tcnt[b + 1]);
    }
  if (lp.tgt_blk.empty()) lp.tgt_off.assign(1, 0);
  lap("contribution sort");
  // block Jacobi scaling targets
  lp.scale_blk.clear();
  for (size_t b = 0; b < pat.bg.size(); ++b)
    if (pat.bg[b] != pat.bh[b] && g.kind[pat.bg[b]] != 0 && g.kind[pat.bh[b]] != 0) lp.scale_blk.push_back((int)b);
  lap("scale blocks");
  // skeleton neighbours + dependency waves (sequential semantics)
  const int nsk = (int)lp.skeleton.size();
  std::vector<int> sk_index(g.G, -1);
  for (int i = 0; i < nsk; ++i) sk_index[lp.skeleton[i]] = i;
  lp.sk_nbr_off.assign(1, 0);
  lp.sk_nbr.clear();
  lp.sk_nbr_blk.clear();
  lp.sk_wave.assign(nsk, 0);
  lp.nwaves = 0;
  for (int i = 0; i < nsk; ++i) {
    const int gg = lp.skeleton[i];
    int w = 0;
    for (int64_t q = pat.adj_off[gg]; q < pat.adj_off[gg + 1]; ++q) {
      const int h = pat.adj_nbr[q];
      if (h == gg || g.kind[h] == 0) continue;
      lp.sk_nbr.push_back(h);
      lp.sk_nbr_blk.push_back(pat.adj_blk[q]);
      const int j = sk_index[h];
      if (j >= 0 && j < i) w = std::max(w, lp.sk_wave[j] + 1);
    }
    lp.sk_nbr_off.push_back((int64_t)lp.sk_nbr.size());
    lp.sk_wave[i] = w;
    lp.nwaves = std::max(lp.nwaves, w + 1);
  }
  lp.sk_ndep.assign(nsk, 0);
  lp.sk_succ_off.assign(nsk + 1, 0);
  for (int i = 0; i < nsk; ++i)
    for (int64_t q = lp.sk_nbr_off[i]; q < lp.sk_nbr_off[i + 1]; ++q) {
      const int j = sk_index[lp.sk_nbr[q]];
      if (j >= 0 && j < i) {
        lp.sk_ndep[i]++;
        lp.sk_succ_off[j + 1]++;
      }
    }
  for (int i = 0; i < nsk; ++i) lp.sk_succ_off[i + 1] += lp.sk_succ_off[i];
  lp.sk_succ.assign(lp.sk_succ_off[nsk], 0);
  {
    std::vector<int64_t> fill(lp.sk_succ_off.begin(), lp.sk_succ_off.end() - 1);
    for (int i = 0; i < nsk; ++i)
      for (int64_t q = lp.sk_nbr_off[i]; q < lp.sk_nbr_off[i + 1]; ++q) {
        const int j = sk_index[lp.sk_nbr[q]];
        if (j >= 0 && j < i) lp.sk_succ[fill[j]++] = i;
      }
  }
  lp.wave_order.resize(nsk);
  std::iota(lp.wave_order.begin(), lp.wave_order.end(), 0);
  std::stable_sort(lp.wave_order.begin(), lp.wave_order.end(),
                   [&](int a, int b) { return lp.sk_wave[a] < lp.sk_wave[b]; });
  lp.wave_off.assign(lp.nwaves + 1, 0);
  for (int i = 0; i < nsk; ++i) lp.wave_off[lp.sk_wave[i] + 1]++;
  for (int w = 0; w < lp.nwaves; ++w) lp.wave_off[w + 1] += lp.wave_off[w];
  lap("skeleton waves");
}

std::string level_json(const LevelPlan& lp) {
  std::ostringstream o;
  o << "{\"level\":" << lp.level << ",\"G\":" << lp.grp.G << ",\"S\":" << lp.grp.mem.size()
    << ",\"p\":" << lp.interior.size() << ",\"q\":" << lp.skeleton.size() << ",\"r\":" << lp.precond.size()
    << ",\"blocks\":" << lp.pat.bg.size() << ",\"pool_doubles\":" << lp.pool_doubles
    << ",\"waves\":" << lp.nwaves << "}";
  return o.str();
}

}  // namespace phif
