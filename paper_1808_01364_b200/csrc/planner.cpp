#include <chrono>
#ifdef _OPENMP
#include <omp.h>
#endif
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
#include <map>
#include <mutex>

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
#pragma omp parallel for schedule(static)
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
  }
  // counting sort of the DOFs by key: per-thread histograms over contiguous DOF ranges keep
  // the members of every key ascending
  int nth = 1;
#ifdef _OPENMP
  nth = omp_get_max_threads();
#endif
  std::vector<std::vector<int>> hist(nth);
  const int64_t chunk = (s.N + nth - 1) / nth;
#pragma omp parallel num_threads(nth)
  {
    int tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
    std::vector<int>& h = hist[tid];
    h.assign(nkeys, 0);
    const int64_t lo = std::min<int64_t>(s.N, tid * chunk), hi = std::min<int64_t>(s.N, lo + chunk);
    for (int64_t i = lo; i < hi; ++i) h[key[i]]++;
  }
  // cnt[k+1] = total of key k; per-thread starts in place of the histograms
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < nkeys; ++k) {
    int64_t t = 0;
    for (int q = 0; q < nth; ++q) t += hist[q][k];
    cnt[k + 1] = t;
  }
  for (int64_t k = 0; k < nkeys; ++k) cnt[k + 1] += cnt[k];
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < nkeys; ++k) {
    int64_t o = cnt[k];
    for (int q = 0; q < nth; ++q) {
      const int v = hist[q][k];
      hist[q][k] = (int)o;
      o += v;
    }
  }
  g.mem.resize(s.N);
#pragma omp parallel num_threads(nth)
  {
    int tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
    std::vector<int>& h = hist[tid];
    const int64_t lo = std::min<int64_t>(s.N, tid * chunk), hi = std::min<int64_t>(s.N, lo + chunk);
    for (int64_t i = lo; i < hi; ++i) g.mem[h[key[i]]++] = (int)i;
  }
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
  const bool tdbg = getenv("PHIF_PLAN_TIMING") != nullptr;
  auto tl = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!tdbg) return;
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "  [classify_next L%d] %-20s %8.2f ms\n", prev.level + 1, what,
            std::chrono::duration<double, std::milli>(now - tl).count());
    tl = now;
  };
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
  lap("survivors + keys");
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
  lap("bucket");
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
  lap("merge members");
  finalize_groups(s, g, {}, gkeys);
  lap("finalize");
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
  // per group: distinct coupled groups h >= g (a per-thread stamp array dedupes in O(1));
  // per-thread lists are concatenated in group order
  int nth = 1;
#ifdef _OPENMP
  nth = omp_get_max_threads();
#endif
  std::vector<std::vector<std::pair<int, int>>> part(nth);
#pragma omp parallel
  {
    int tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
    std::vector<std::pair<int, int>>& mine = part[tid];
    mine.reserve((size_t)(N / nth + 1) * 4);
    std::vector<int> stamp(g.G, -1);
#pragma omp for schedule(static)
    for (int i = 0; i < g.G; ++i) {
      for (int64_t p = g.off[i]; p < g.off[i + 1]; ++p) {
        const int r = g.mem[p];
        for (int64_t e = rowptr[r]; e < rowptr[r + 1]; ++e) {
          const int h = gid[col[e]];
          if (h >= i && stamp[h] != i) {
            stamp[h] = i;
            mine.emplace_back(i, h);
          }
        }
      }
    }
  }
  std::vector<std::pair<int, int>> pairs;
  size_t tot = 0;
  for (auto& v : part) tot += v.size();
  pairs.reserve(tot);
  for (auto& v : part) pairs.insert(pairs.end(), v.begin(), v.end());
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
  // per-thread lists over block ranges, concatenated (build_level sorts and dedups per group)
  const int64_t nb = (int64_t)prev.pat.bg.size();
  int nth = 1;
#ifdef _OPENMP
  nth = omp_get_max_threads();
#endif
  std::vector<std::vector<std::pair<int, int>>> part(nth);
#pragma omp parallel num_threads(nth)
  {
    int tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
    std::vector<std::pair<int, int>>& mine = part[tid];
    const int64_t lo = nb * tid / nth, hi = nb * (tid + 1) / nth;
    mine.reserve(hi - lo);
    for (int64_t b = lo; b < hi; ++b) {
      const int og = prev.pat.bg[b], oh = prev.pat.bh[b];
      if (prev.grp.kind[og] == 0 || prev.grp.kind[oh] == 0) continue;
      const int G = old2new[og], H = old2new[oh];
      if (G < 0 || H < 0) continue;
      mine.emplace_back(std::min(G, H), std::max(G, H));
    }
  }
  std::vector<std::pair<int, int>> pairs;
  size_t tot = 0;
  for (auto& v : part) tot += v.size();
  pairs.reserve(tot);
  for (auto& v : part) pairs.insert(pairs.end(), v.begin(), v.end());
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
// Stable parallel counting sort: item i in [0, n) has key(i) in [0, K) (or < 0: dropped). Fills
// off (K+1) and calls emit(i, pos) with the item's position in key order (stable in i). Per-thread
// histograms over contiguous item ranges.
template <class KeyF, class EmitF>
static void par_bucket(int64_t n, int K, KeyF key, std::vector<int64_t>& off, EmitF emit) {
  int nth = 1;
#ifdef _OPENMP
  nth = omp_get_max_threads();
#endif
  const int64_t chunk = (n + nth - 1) / nth;
  std::vector<std::vector<int64_t>> hist(nth);
  off.assign((size_t)K + 1, 0);
#pragma omp parallel num_threads(nth)
  {
    int tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
    std::vector<int64_t>& h = hist[tid];
    h.assign(K, 0);
    const int64_t lo = std::min<int64_t>(n, tid * chunk), hi = std::min<int64_t>(n, lo + chunk);
    for (int64_t i = lo; i < hi; ++i) {
      const int k = key(i);
      if (k >= 0) h[k]++;
    }
#pragma omp barrier
#pragma omp for schedule(static)
    for (int k = 0; k < K; ++k) {
      int64_t t = 0;
      for (int q = 0; q < nth; ++q) t += hist[q][k];
      off[k + 1] = t;
    }
#pragma omp single
    for (int k = 0; k < K; ++k) off[k + 1] += off[k];
#pragma omp for schedule(static)
    for (int k = 0; k < K; ++k) {
      int64_t o = off[k];
      for (int q = 0; q < nth; ++q) {
        const int64_t v = hist[q][k];
        hist[q][k] = o;
        o += v;
      }
    }
    for (int64_t i = lo; i < hi; ++i) {
      const int k = key(i);
      if (k >= 0) emit(i, h[k]++);
    }
  }
}

static void upper_lists(int G, const std::vector<std::pair<int, int>>& pairs, std::vector<int64_t>& off,
                        std::vector<int>& nbr) {
  nbr.assign(pairs.size(), 0);
  par_bucket((int64_t)pairs.size(), G, [&](int64_t i) { return pairs[i].first; }, off,
             [&](int64_t i, int64_t pos) { nbr[pos] = pairs[i].second; });
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
#pragma omp parallel for schedule(static)
  for (int gi = 0; gi < G; ++gi)
    for (int64_t q = uoff[gi]; q < uoff[gi + 1]; ++q) {
      pat.bg[q] = gi;
      pat.bh[q] = unbr[q];
    }
  // lower neighbours of h (blocks (g, h), g < h), in increasing g: stable bucket of the blocks by h
  std::vector<int64_t> loff;
  std::vector<int64_t> lpos(nb, -1);
  par_bucket(nb, G, [&](int64_t q) { return unbr[q] != pat.bg[q] ? unbr[q] : -1; }, loff,
             [&](int64_t q, int64_t pos) { lpos[q] = pos; });
  pat.adj_off.assign(G + 1, 0);
  for (int gi = 0; gi < G; ++gi) pat.adj_off[gi + 1] = loff[gi + 1] + uoff[gi + 1];
  pat.adj_nbr.assign(pat.adj_off[G], 0);
  pat.adj_blk.assign(pat.adj_off[G], 0);
#pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < nb; ++q)
    if (lpos[q] >= 0) {
      const int h = unbr[q];
      const int64_t f = pat.adj_off[h] + (lpos[q] - loff[h]);
      pat.adj_nbr[f] = pat.bg[q];
      pat.adj_blk[f] = (int)q;
    }
#pragma omp parallel for schedule(static)
  for (int gi = 0; gi < G; ++gi) {
    int64_t f = pat.adj_off[gi] + (loff[gi + 1] - loff[gi]);
    for (int64_t q = uoff[gi]; q < uoff[gi + 1]; ++q) {
      pat.adj_nbr[f] = unbr[q];
      pat.adj_blk[f++] = (int)q;
    }
  }
}

// exclusive prefix of per-item counts (serial; the counts are computed in parallel)
static int64_t prefix_counts(std::vector<int64_t>& off) {
  int64_t acc = 0;
  for (size_t i = 0; i + 1 < off.size(); ++i) {
    const int64_t v = off[i + 1];
    off[i + 1] = acc + v;
    acc += v;
  }
  return acc;
}

void build_level(const Spec& s, LevelPlan& lp, std::vector<std::pair<int, int>> pairs) {
  const bool tdbg = getenv("PHIF_PLAN_TIMING") != nullptr;
  auto tl = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!tdbg) return;
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "  [plan L%d] %-28s %8.2f ms\n", lp.grp.level, what,
            std::chrono::duration<double, std::milli>(now - tl).count());
    tl = now;
  };
  Groups& g = lp.grp;
  const int G = g.G;
  lp.level = g.level;
  lp.root = (g.level == s.L);
  for (int i = 0; i < G; ++i) pairs.emplace_back(i, i);
  std::vector<int64_t> uoff;
  std::vector<int> unbr;
  upper_lists(G, pairs, uoff, unbr);
  std::vector<std::pair<int, int>>().swap(pairs);
  lap("stencil upper lists");
  lp.interior.clear();
  lp.precond.clear();
  lp.skeleton.clear();
  for (int i = 0; i < G; ++i) {
    if (g.kind[i] == 0) {
      lp.interior.push_back(i);
    } else {
      lp.precond.push_back(i);
      if (g.kind[i] == 1) lp.skeleton.push_back(i);
    }
  }
  // an interior group is the first group of its cell closure: every coupling of it is an upper entry
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(max : bad)
  for (int gi = 0; gi < G; ++gi)
    for (int64_t q = uoff[gi]; q < uoff[gi + 1]; ++q)
      if (unbr[q] != gi && g.kind[unbr[q]] == 0) bad = std::max(bad, g.kind[gi] == 0 ? 2 : 1);
  if (bad == 2) throw std::runtime_error("planner: two interior groups coupled");
  if (bad == 1) throw std::runtime_error("planner: interior group is not first in its closure");
  lap("classify + checks");
  // cells of every boundary group (interiors in cell order)
  const int p = (int)lp.interior.size();
  std::vector<int64_t> roff(G + 1, 0);
  for (int t = 0; t < p; ++t) {
    const int I = lp.interior[t];
    for (int64_t q = uoff[I]; q < uoff[I + 1]; ++q)
      if (unbr[q] != I) roff[unbr[q] + 1]++;
  }
  for (int i = 0; i < G; ++i) roff[i + 1] += roff[i];
  std::vector<int> rcell(roff[G]);
  {
    std::vector<int64_t> fill(roff.begin(), roff.end() - 1);
    for (int t = 0; t < p; ++t) {
      const int I = lp.interior[t];
      for (int64_t q = uoff[I]; q < uoff[I + 1]; ++q)
        if (unbr[q] != I) rcell[fill[unbr[q]]++] = t;
    }
  }
  // block pattern after elimination fill: upper(g) = stencil upper(g) plus every
  // h >= g sharing a cell with g; two passes (count, fill), groups in parallel
  std::vector<int64_t> foff(G + 1, 0);
  std::vector<int> fnbr;
  for (int pass = 0; pass < 2; ++pass) {
#pragma omp parallel
    {
      std::vector<int> buf;
#pragma omp for schedule(dynamic, 256)
      for (int gi = 0; gi < G; ++gi) {
        buf.assign(unbr.begin() + uoff[gi], unbr.begin() + uoff[gi + 1]);
        for (int64_t e = roff[gi]; e < roff[gi + 1]; ++e) {
          const int I = lp.interior[rcell[e]];
          for (int64_t q = uoff[I]; q < uoff[I + 1]; ++q)
            if (unbr[q] >= gi && unbr[q] != I) buf.push_back(unbr[q]);
        }
        std::sort(buf.begin(), buf.end());
        const int64_t nu = std::unique(buf.begin(), buf.end()) - buf.begin();
        if (pass == 0) foff[gi + 1] = nu;
        else std::copy(buf.begin(), buf.begin() + nu, fnbr.begin() + foff[gi]);
      }
    }
    if (pass == 0) fnbr.assign(prefix_counts(foff), 0);
  }
  uoff.swap(foff);
  unbr.swap(fnbr);
  lap("fill pattern");
  adjacency_from_upper(G, uoff, unbr, lp.pat);
  const Pattern& pat = lp.pat;
  const int64_t nblocks = (int64_t)pat.bg.size();
  lap("adjacency");
  // pool
  lp.boff.resize(nblocks);
  {
    int nth = 1;
#ifdef _OPENMP
    nth = omp_get_max_threads();
#endif
    std::vector<int64_t> part(nth + 1, 0);
    const int64_t ch = (nblocks + nth - 1) / nth;
#pragma omp parallel num_threads(nth)
    {
      int tid = 0;
#ifdef _OPENMP
      tid = omp_get_thread_num();
#endif
      const int64_t lo = std::min<int64_t>(nblocks, tid * ch), hi = std::min<int64_t>(nblocks, lo + ch);
      int64_t a = 0;
      for (int64_t b = lo; b < hi; ++b) {
        lp.boff[b] = a;
        a += (int64_t)g.size(pat.bg[b]) * g.size(pat.bh[b]);
      }
      part[tid + 1] = a;
#pragma omp barrier
#pragma omp single
      for (int q = 0; q < nth; ++q) part[q + 1] += part[q];
      for (int64_t b = lo; b < hi; ++b) lp.boff[b] += part[tid];
    }
    lp.pool_doubles = part[nth];
  }
  lap("pool");
  // cells: boundary = neighbour groups of I (all after I)
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
  }
  // Schur targets: block (a, b), a <= b, receives U_t[a, b] from every cell t holding both a and b
  // (cells of a intersect cells of b; both lists ascending in cell order = the summation order)
  auto pos_in_cell = [&](int t, int h) {   // index of group h in cell t's neighbour list
    const int* b0 = lp.cell_nbr.data() + lp.cell_nbr_off[t];
    const int* b1 = lp.cell_nbr.data() + lp.cell_nbr_off[t + 1];
    return (int)(std::lower_bound(b0, b1, h) - b0);
  };
  auto col_of = [&](int t, int h) {   // first column of group h in cell t's boundary
    const int* b0 = lp.cell_nbr.data() + lp.cell_nbr_off[t];
    const int* b1 = lp.cell_nbr.data() + lp.cell_nbr_off[t + 1];
    return lp.cell_nbr_col[lp.cell_nbr_off[t] + (std::lower_bound(b0, b1, h) - b0)];
  };
  std::vector<int64_t> tcnt(nblocks + 1, 0);
  for (int pass = 0; pass < 2; ++pass) {
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t b = 0; b < nblocks; ++b) {
      const int a0 = pat.bg[b], b0 = pat.bh[b];
      if (g.kind[a0] == 0 || g.kind[b0] == 0) {
        if (pass == 0) tcnt[b + 1] = 0;
        continue;
      }
      int64_t o = pass ? tcnt[b] : 0;
      int64_t ia = roff[a0], ib = roff[b0];
      const int64_t ea = roff[a0 + 1], eb = roff[b0 + 1];
      while (ia < ea && ib < eb) {
        if (rcell[ia] < rcell[ib]) {
          ++ia;
        } else if (rcell[ib] < rcell[ia]) {
          ++ib;
        } else {
          if (pass) {
            const int t = rcell[ia];
            lp.con_cell[o] = t;
            lp.con_row[o] = col_of(t, a0);
            lp.con_col[o] = col_of(t, b0);
            lp.con_ri[o] = pos_in_cell(t, a0);
            lp.con_ci[o] = pos_in_cell(t, b0);
          }
          ++o;
          ++ia;
          ++ib;
        }
      }
      if (pass == 0) tcnt[b + 1] = o;
    }
    if (pass == 0) {
      const int64_t ncons = prefix_counts(tcnt);
      lp.con_cell.resize(ncons);
      lp.con_row.resize(ncons);
      lp.con_col.resize(ncons);
      lp.con_ri.resize(ncons);
      lp.con_ci.resize(ncons);
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
  lap("cells + Schur targets");
  // block Jacobi scaling targets
  lp.scale_blk.clear();
  for (int64_t b = 0; b < nblocks; ++b)
    if (pat.bg[b] != pat.bh[b] && g.kind[pat.bg[b]] != 0 && g.kind[pat.bh[b]] != 0) lp.scale_blk.push_back((int)b);
  lap("scale blocks");
  // skeleton neighbours + dependency waves (sequential semantics)
  const int nsk = (int)lp.skeleton.size();
  std::vector<int> sk_index(G, -1);
  for (int i = 0; i < nsk; ++i) sk_index[lp.skeleton[i]] = i;
  lp.sk_nbr_off.assign(nsk + 1, 0);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < nsk; ++i) {
    const int gg = lp.skeleton[i];
    int64_t cnt = 0;
    for (int64_t q = pat.adj_off[gg]; q < pat.adj_off[gg + 1]; ++q) {
      const int h = pat.adj_nbr[q];
      if (h != gg && g.kind[h] != 0) ++cnt;
    }
    lp.sk_nbr_off[i + 1] = cnt;
  }
  lp.sk_nbr.assign(prefix_counts(lp.sk_nbr_off), 0);
  lp.sk_nbr_blk.assign(lp.sk_nbr.size(), 0);
  lp.sk_ndep.assign(nsk, 0);
  lp.sk_succ_off.assign(nsk + 1, 0);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < nsk; ++i) {
    const int gg = lp.skeleton[i];
    int64_t o = lp.sk_nbr_off[i];
    int nd = 0, ns = 0;
    for (int64_t q = pat.adj_off[gg]; q < pat.adj_off[gg + 1]; ++q) {
      const int h = pat.adj_nbr[q];
      if (h == gg || g.kind[h] == 0) continue;
      lp.sk_nbr[o] = h;
      lp.sk_nbr_blk[o++] = pat.adj_blk[q];
      const int j = sk_index[h];
      if (j >= 0 && j < i) ++nd;
      if (j > i) ++ns;
    }
    lp.sk_ndep[i] = nd;
    lp.sk_succ_off[i + 1] = ns;
  }
  // later coupled separators (the adjacency is symmetric); waves: 1 + latest earlier neighbour
  lp.sk_succ.assign(prefix_counts(lp.sk_succ_off), 0);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < nsk; ++i) {
    int64_t o = lp.sk_succ_off[i];
    for (int64_t q = lp.sk_nbr_off[i]; q < lp.sk_nbr_off[i + 1]; ++q) {
      const int j = sk_index[lp.sk_nbr[q]];
      if (j > i) lp.sk_succ[o++] = j;
    }
  }
  lp.sk_wave.assign(nsk, 0);
  lp.nwaves = 0;
  for (int i = 0; i < nsk; ++i) {
    int w = 0;
    for (int64_t q = lp.sk_nbr_off[i]; q < lp.sk_nbr_off[i + 1]; ++q) {
      const int j = sk_index[lp.sk_nbr[q]];
      if (j >= 0 && j < i) w = std::max(w, lp.sk_wave[j] + 1);
    }
    lp.sk_wave[i] = w;
    lp.nwaves = std::max(lp.nwaves, w + 1);
  }
  lp.wave_off.assign(lp.nwaves + 1, 0);
  for (int i = 0; i < nsk; ++i) lp.wave_off[lp.sk_wave[i] + 1]++;
  for (int w = 0; w < lp.nwaves; ++w) lp.wave_off[w + 1] += lp.wave_off[w];
  lp.wave_order.resize(nsk);
  {
    std::vector<int64_t> fill(lp.wave_off.begin(), lp.wave_off.end() - 1);
    for (int i = 0; i < nsk; ++i) lp.wave_order[fill[lp.sk_wave[i]]++] = i;   // stable: (wave, index)
  }
  lap("skeleton waves");
}

namespace {
template <class T>
struct VecPool {
  std::mutex mu;
  std::multimap<size_t, std::vector<T>> free;   // by capacity
  size_t bytes = 0;
  static constexpr size_t CAP = (size_t)2 << 30;   // keep at most 2 GB of host plan arrays
  std::vector<T> take(size_t n) {
    {
      std::lock_guard<std::mutex> lock(mu);
      auto it = free.lower_bound(n);
      if (it != free.end() && it->first <= 2 * n + 4096) {
        std::vector<T> v = std::move(it->second);
        bytes -= it->first * sizeof(T);
        free.erase(it);
        v.resize(n);   // truncation, or a short zero tail
        return v;
      }
    }
    return std::vector<T>(n);
  }
  void give(std::vector<T>& v) {
    if (v.capacity() < 4096) return;
    std::vector<T> w;
    w.swap(v);
    std::lock_guard<std::mutex> lock(mu);
    if (bytes + w.capacity() * sizeof(T) > CAP) return;
    bytes += w.capacity() * sizeof(T);
    free.emplace(w.capacity(), std::move(w));
  }
};
VecPool<int>& ipool() {
  static VecPool<int>* p = new VecPool<int>();
  return *p;
}
VecPool<int64_t>& lpool() {
  static VecPool<int64_t>* p = new VecPool<int64_t>();
  return *p;
}
}  // namespace

std::vector<int> pool_take_int(size_t n) { return ipool().take(n); }
std::vector<int64_t> pool_take_i64(size_t n) { return lpool().take(n); }

void recycle_plan(LevelPlan& lp) {
  for (std::vector<int>* v : {&lp.grp.q, &lp.grp.bits, &lp.grp.kind, &lp.grp.mem, &lp.grp.src_group, &lp.grp.src_pos,
                              &lp.grp.src_local, &lp.grp.srcl, &lp.pat.bg, &lp.pat.bh, &lp.pat.adj_nbr,
                              &lp.pat.adj_blk, &lp.interior, &lp.precond, &lp.skeleton, &lp.cell_nbr,
                              &lp.cell_nbr_blk, &lp.cell_nbr_col, &lp.cell_n, &lp.cell_b, &lp.tgt_blk, &lp.con_cell,
                              &lp.con_row, &lp.con_col, &lp.con_ri, &lp.con_ci, &lp.scale_blk, &lp.sk_nbr, &lp.sk_nbr_blk, &lp.sk_wave,
                              &lp.wave_order, &lp.sk_ndep, &lp.sk_succ})
    ipool().give(*v);
  for (std::vector<int64_t>* v : {&lp.grp.off, &lp.grp.srcl_off, &lp.pat.adj_off, &lp.boff, &lp.cell_nbr_off,
                                  &lp.tgt_off, &lp.sk_nbr_off, &lp.wave_off, &lp.sk_succ_off})
    lpool().give(*v);
}

LevelPlan preplan_next(const Spec& s, const LevelPlan& prev) {
  const Groups& pg = prev.grp;
  std::vector<uint8_t> alive(pg.mem.size(), 0);
#pragma omp parallel for schedule(static)
  for (int g = 0; g < pg.G; ++g)
    if (pg.kind[g] != 0)
      for (int64_t q = pg.off[g]; q < pg.off[g + 1]; ++q) alive[q] = 1;
  LevelPlan lp;
  lp.grp = classify_next(s, pg, alive);
  build_level(s, lp, pattern_next(prev, lp.grp));
  return lp;
}

bool finish_preplan(const Spec& s, LevelPlan& lp, const LevelPlan& prev, const std::vector<uint8_t>& alive) {
  (void)s;
  Groups& g = lp.grp;
  const Groups& pg = prev.grp;
  const int G = g.G;
  // every non-interior old group must keep a DOF (else the grouping differs)
  int lost = 0;
#pragma omp parallel for schedule(static) reduction(max : lost)
  for (int og = 0; og < pg.G; ++og) {
    if (pg.kind[og] == 0) continue;
    bool any = false;
    for (int64_t q = pg.off[og]; q < pg.off[og + 1] && !any; ++q) any = alive[q] != 0;
    if (!any) lost = 1;
  }
  if (lost) return false;
  // filtered member lists (survivors keep their ascending order and provenance)
  // (arrays from the host pool: recycled allocations, no fresh page faults on this path)
  std::vector<int64_t> cnt = pool_take_i64((size_t)G + 1);
  cnt[0] = 0;
#pragma omp parallel for schedule(dynamic, 256)
  for (int i = 0; i < G; ++i) {
    int64_t c = 0;
    for (int64_t q = g.off[i]; q < g.off[i + 1]; ++q) c += alive[pg.off[g.src_group[q]] + g.src_pos[q]] != 0;
    cnt[i + 1] = c;
  }
  for (int i = 0; i < G; ++i) cnt[i + 1] += cnt[i];
  const int64_t tot = cnt[G];
  std::vector<int> mem = pool_take_int(tot), sg = pool_take_int(tot), sp = pool_take_int(tot), sl = pool_take_int(tot);
#pragma omp parallel for schedule(dynamic, 256)
  for (int i = 0; i < G; ++i) {
    int64_t o = cnt[i];
    for (int64_t q = g.off[i]; q < g.off[i + 1]; ++q)
      if (alive[pg.off[g.src_group[q]] + g.src_pos[q]]) {
        mem[o] = g.mem[q];
        sg[o] = g.src_group[q];
        sp[o] = g.src_pos[q];
        sl[o] = g.src_local[q];
        ++o;
      }
  }
  g.off.swap(cnt);
  g.mem.swap(mem);
  g.src_group.swap(sg);
  g.src_pos.swap(sp);
  g.src_local.swap(sl);
  lpool().give(cnt);
  ipool().give(mem);
  ipool().give(sg);
  ipool().give(sp);
  ipool().give(sl);
  // size-dependent parts of the plan
  const int64_t nb = (int64_t)lp.pat.bg.size();
  {
    int64_t acc = 0;
    for (int64_t b = 0; b < nb; ++b) {
      lp.boff[b] = acc;
      acc += (int64_t)g.size(lp.pat.bg[b]) * g.size(lp.pat.bh[b]);
    }
    lp.pool_doubles = acc;
  }
  const int p = (int)lp.interior.size();
#pragma omp parallel for schedule(static)
  for (int t = 0; t < p; ++t) {
    int bc = 0;
    for (int64_t j = lp.cell_nbr_off[t]; j < lp.cell_nbr_off[t + 1]; ++j) {
      lp.cell_nbr_col[j] = bc;
      bc += g.size(lp.cell_nbr[j]);
    }
    lp.cell_n[t] = g.size(lp.interior[t]);
    lp.cell_b[t] = bc;
  }
  const int64_t ncon = (int64_t)lp.con_cell.size();
#pragma omp parallel for schedule(static)
  for (int64_t o = 0; o < ncon; ++o) {
    const int64_t base = lp.cell_nbr_off[lp.con_cell[o]];
    lp.con_row[o] = lp.cell_nbr_col[base + lp.con_ri[o]];
    lp.con_col[o] = lp.cell_nbr_col[base + lp.con_ci[o]];
  }
  return true;
}

void compute_waves(LevelPlan& lp, int G) {
  const int nsk = (int)lp.skeleton.size();
  std::vector<int> ski(G, -1);
  for (int i = 0; i < nsk; ++i) ski[lp.skeleton[i]] = i;
  lp.sk_wave.assign(nsk, 0);
  lp.nwaves = 0;
  for (int i = 0; i < nsk; ++i) {
    int w = 0;
    for (int64_t q = lp.sk_nbr_off[i]; q < lp.sk_nbr_off[i + 1]; ++q) {
      const int j = ski[lp.sk_nbr[q]];
      if (j >= 0 && j < i) w = std::max(w, lp.sk_wave[j] + 1);
    }
    lp.sk_wave[i] = w;
    lp.nwaves = std::max(lp.nwaves, w + 1);
  }
  lp.wave_off.assign(lp.nwaves + 1, 0);
  for (int i = 0; i < nsk; ++i) lp.wave_off[lp.sk_wave[i] + 1]++;
  for (int w = 0; w < lp.nwaves; ++w) lp.wave_off[w + 1] += lp.wave_off[w];
  lp.wave_order.resize(nsk);
  std::vector<int64_t> fill(lp.wave_off.begin(), lp.wave_off.end() - 1);
  for (int i = 0; i < nsk; ++i) lp.wave_order[fill[lp.sk_wave[i]]++] = i;   // stable: (wave, index)
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
