#include <future>
#include <omp.h>
#include <mutex>
#include <numeric>
// Host driver: per level plan -> device structures -> batched stage launches.
//
// factorize() restates SPEC.md:275-283 (level loop, root Cholesky as the level-L
// elimination), apply() SPEC.md:293-310 (record replay), pcg() SPEC.md:360-378,
// solve_error() SPEC.md:418-426 (e_s in the symmetric G-congruence form).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <numeric>
#include <sstream>

#include "engine.h"
#include "gpu_plan.h"
#include "problem.h"

namespace phif {

// cells / groups / separators with at least this many DOFs take the tile-parallel paths
// (PHIF_BIG_CELL / PHIF_BIG_PREC / PHIF_BIG_SEP override, for tuning)
static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}
static const int BIG_CELL = env_int("PHIF_BIG_CELL", 64);
static const int BIG_PREC = env_int("PHIF_BIG_PREC", 64);
static const int BIG_SEP = env_int("PHIF_BIG_SEP", 192);
constexpr int APPLY_BIG = 96;    // groups with |g| >= APPLY_BIG are replayed by batched GEMMs

static std::chrono::steady_clock::time_point g_dbg_t0 = std::chrono::steady_clock::now();
static double dbg_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - g_dbg_t0).count();
}
static bool debug_on() {
  static int on = -1;
  if (on < 0) on = getenv("PHIF_DEBUG") ? 1 : 0;
  return on == 1;
}
#define DBG(...)                                  \
  do {                                            \
    if (debug_on()) {                             \
      fprintf(stderr, "[phif %9.2f] ", dbg_ms());  \
      fprintf(stderr, __VA_ARGS__);               \
      fprintf(stderr, "\n");                      \
      fflush(stderr);                             \
    }                                             \
  } while (0)

#define CK(x)                                                                                    \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess) throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));    \
  } while (0)

DBuf& DBuf::operator=(DBuf&& o) noexcept {
  if (this != &o) {
    release();
    p = o.p;
    bytes = o.bytes;
    s = o.s;
    o.p = nullptr;
    o.bytes = 0;
  }
  return *this;
}

// Caching device allocator: blocks come from cudaMalloc once and are recycled by size class
// (never returned to the driver). Thread-safe (one mutex) and stream-ordered: a block released on
// stream s carries an event recorded on s at release; a later request from the same stream reuses
// it directly (stream order already serialises the old and the new user), a request from another
// stream first makes that stream wait on the event (no host synchronisation either way).
namespace {
struct DeviceCache {
  struct Blk {
    void* p;
    cudaStream_t s;
    cudaEvent_t ev;
    int dev;
  };
  std::multimap<size_t, Blk> free_blocks;
  std::vector<cudaEvent_t> events;   // recycled release events
  size_t cached = 0;
  std::mutex mu;
  static size_t round(size_t b) {
    if (b <= (1u << 20)) return (b + 511) & ~size_t(511);
    return (b + (size_t(2) << 20) - 1) & ~((size_t(2) << 20) - 1);
  }
  void* get(size_t& b, cudaStream_t st) {
    b = round(b);
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    // best fit within +25%, preferring a block released on the requesting stream
    auto lo = free_blocks.lower_bound(b), hi = free_blocks.upper_bound(b + b / 4);
    auto pick = free_blocks.end();
    for (auto it = lo; it != hi; ++it) {
      if (it->second.dev != dev) continue;
      if (it->second.s == st) {
        pick = it;
        break;
      }
      if (pick == free_blocks.end()) pick = it;
    }
    if (pick != free_blocks.end()) {
      Blk k = pick->second;
      b = pick->first;
      cached -= b;
      free_blocks.erase(pick);
      if (k.s != st) CK(cudaStreamWaitEvent(st, k.ev, 0));
      events.push_back(k.ev);
      return k.p;
    }
    void* p = nullptr;
    if (cudaMalloc(&p, b) != cudaSuccess) {
      cudaGetLastError();
      // release the cached blocks of this device (after their last users) and retry once
      for (auto it = free_blocks.begin(); it != free_blocks.end();) {
        if (it->second.dev == dev) {
          cudaEventSynchronize(it->second.ev);
          cudaFree(it->second.p);
          events.push_back(it->second.ev);
          cached -= it->first;
          it = free_blocks.erase(it);
        } else {
          ++it;
        }
      }
      CK(cudaMalloc(&p, b));
    }
    return p;
  }
  void put(void* p, size_t b, cudaStream_t st) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    cudaEvent_t ev;
    if (events.empty()) {
      CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    } else {
      ev = events.back();
      events.pop_back();
    }
    if (cudaEventRecord(ev, st) != cudaSuccess) {   // (stream already destroyed: order on the device)
      cudaGetLastError();
      cudaDeviceSynchronize();
      CK(cudaEventRecord(ev, 0));
    }
    free_blocks.emplace(b, Blk{p, st, ev, dev});
    cached += b;
  }
};
DeviceCache& dcache() {
  static DeviceCache* c = new DeviceCache();   // intentionally leaked: outlives static destructors
  return *c;
}
}  // namespace

void DBuf::alloc(size_t nbytes, cudaStream_t st, bool zero) {
  release();
  s = st;
  bytes = std::max<size_t>(nbytes, 8);
  p = dcache().get(bytes, st);
  if (zero) CK(cudaMemsetAsync(p, 0, bytes, st));
}

void DBuf::release() {
  if (p) dcache().put(p, bytes, s);
  p = nullptr;
  bytes = 0;
}

LevelDev LevelRT::dev() const {
  LevelDev d;
  d.G = plan.grp.G;
  d.goff = goff.as<int64_t>();
  d.mem = mem.as<int>();
  d.gsize = gsize.as<int>();
  d.pool = pool.as<double>();
  d.boff = boff.as<int64_t>();
  d.bg = bg.as<int>();
  d.bh = bh.as<int>();
  d.adj_off = adj_off.as<int64_t>();
  d.adj_nbr = adj_nbr.as<int>();
  d.adj_blk = adj_blk.as<int>();
  d.diag_blk = diag_blk.as<int>();
  return d;
}

std::unique_ptr<Matrix> matrix_create(const int64_t* rowptr, const int* col, const double* val, int64_t N,
                                      cudaStream_t s) {
  auto A = std::make_unique<Matrix>();
  A->N = N;
  A->nnz = rowptr[N];
  // host copies of the pattern for the planner (parallel chunked copies; a few threads saturate
  // the host memory bandwidth)
  A->h_rowptr.reset(new int64_t[N + 1]);
  A->h_col.reset(new int[std::max<int64_t>(A->nnz, 1)]);
  auto pcopy = [](void* dst, const void* src, size_t bytes) {
    const int64_t nchunk = (int64_t)std::max<size_t>(1, bytes >> 22);
#pragma omp parallel for schedule(dynamic, 1) num_threads(std::min<int64_t>(nchunk, 6))
    for (int64_t c = 0; c < nchunk; ++c) {
      const size_t a = bytes * c / nchunk, e = bytes * (c + 1) / nchunk;
      memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, e - a);
    }
  };
  pcopy(A->h_rowptr.get(), rowptr, (N + 1) * sizeof(int64_t));
  pcopy(A->h_col.get(), col, A->nnz * sizeof(int));
  A->rowptr.alloc((N + 1) * sizeof(int64_t), s);
  A->col.alloc(A->nnz * sizeof(int), s);
  A->val.alloc(A->nnz * sizeof(double), s);
  upload_bytes(A->rowptr.p, rowptr, (N + 1) * sizeof(int64_t), s);
  upload_bytes(A->col.p, col, A->nnz * sizeof(int), s);
  upload_bytes(A->val.p, val, A->nnz * sizeof(double), s);
  return A;
}

void Matrix::ensure_host_pattern(cudaStream_t s) const {
  if (h_rowptr) return;
  h_rowptr.reset(new int64_t[N + 1]);
  h_col.reset(new int[std::max<int64_t>(nnz, 1)]);
  download_bytes(h_rowptr.get(), rowptr.p, (N + 1) * sizeof(int64_t), s);
  download_bytes(h_col.get(), col.p, nnz * sizeof(int), s);
}

namespace {

using clk = std::chrono::steady_clock;
double ms_since(clk::time_point t0) {
  return std::chrono::duration<double, std::milli>(clk::now() - t0).count();
}

void check_status(Factorization& F, int level, int stage) {
  DevStatus h;
  CK(cudaMemcpyAsync(&h, F.status.p, sizeof(h), cudaMemcpyDeviceToHost, F.stream));
  CK(cudaStreamSynchronize(F.stream));
  CK(cudaGetLastError());
  if (h.first_bad != ~0ull) {
    const int op = (int)(h.first_bad >> 32), piv = (int)(h.first_bad & 0xffffffffu);
    throw NotSpd(piv, level, stage, op);
  }
}

void upload_structure(LevelRT& L, cudaStream_t s) {
  const LevelPlan& p = L.plan;
  const Groups& g = p.grp;
  upload(L.goff, g.off, s);
  upload(L.mem, g.mem, s);
  std::vector<int> gs(g.G);
  for (int i = 0; i < g.G; ++i) gs[i] = g.size(i);
  upload(L.gsize, gs, s);
  upload(L.boff, p.boff, s);
  upload(L.bg, p.pat.bg, s);
  upload(L.bh, p.pat.bh, s);
  upload(L.adj_off, p.pat.adj_off, s);
  upload(L.adj_nbr, p.pat.adj_nbr, s);
  upload(L.adj_blk, p.pat.adj_blk, s);
  std::vector<int> diag(g.G, -1);
  for (size_t b = 0; b < p.pat.bg.size(); ++b)
    if (p.pat.bg[b] == p.pat.bh[b]) diag[p.pat.bg[b]] = (int)b;
  upload(L.diag_blk, diag, s);
}

// Work lists for the tile-parallel big-cell path (one level).
struct BigPlan {
  // Right-looking blocked Cholesky of the big panels, all big cells of the level together.
  // Blocks of KB columns; inside a block, 64-wide steps (diag factor + inverse, panel TRSM as a
  // GEMM with the inverse, update of the block's own remaining columns); then one KB-deep
  // update of the whole trailing matrix. Last, U = X^T X (lower tiles, mirrored).
  static constexpr int T = 64;
  const int KB = env_int("PHIF_BIG_KB", 256);   // multiple of 128
  const bool wide128 = env_int("PHIF_WIDE128", 0) != 0;   // (measured: no gain over the 64-tile kernel)
  DBuf d_n, d_b, d_rows, d_P, d_U, d_op, d_linv, d_list;
  DBuf d_cell, d_i, d_j;
  struct Phase {
    int kind;        // 0 diag + trsm + narrow update (one 64-wide step), 1 wide update of the next
                     // block's columns, 3 wide update beyond the next block (side stream), 2 U
    int64_t off[3], cnt[3];
    int k0, kw;
  };
  std::vector<Phase> phases;
  int nbig = 0;
  int64_t nwork_total = 0;
  void build(const std::vector<int>& big, const std::vector<int>& cn, const std::vector<int>& cb, double* rec,
             const std::vector<int64_t>& P_off, double* U, const std::vector<int64_t>& U_off, cudaStream_t s) {
    nbig = (int)big.size();
    std::vector<int> n(nbig), b(nbig), op(nbig), rws(nbig);
    std::vector<double*> Pp(nbig), Up(nbig);
    int nmax = 0;
    for (int c = 0; c < nbig; ++c) {
      const int t = big[c];
      n[c] = cn[t];
      b[c] = cb[t];
      op[c] = t;
      rws[c] = n[c] + b[c] + n[c];
      Pp[c] = rec + P_off[t];
      Up[c] = U + U_off[t];
      nmax = std::max(nmax, n[c]);
    }
    std::vector<int> wc, wi, wj;
    // trailing tiles of cell c for columns [base, cend), rows [base, rows): skip tiles strictly
    // above the diagonal of the square part
    // Identity row i (panel row n+b+i) holds nonzeros only in columns >= i (it becomes row i of
    // L^-T), so its update from the K range [.., kend) vanishes when i >= kend: such tiles are
    // skipped (zero_tile).
    auto zero_tile = [&](int c, int r0, int kend) { return r0 - (n[c] + b[c]) >= kend; };
    auto trailing = [&](int c, int base, int cend, int kend, int T = BigPlan::T) {
      if (base >= cend) return;
      const int nr = (rws[c] - base + T - 1) / T, nc = (cend - base + T - 1) / T;
      for (int it = 0; it < nr; ++it)
        for (int jt = 0; jt < nc; ++jt) {
          if (jt > it && base + T * (it + 1) <= n[c]) continue;
          if (zero_tile(c, base + T * it, kend)) continue;
          wc.push_back(c);
          wi.push_back(it);
          wj.push_back(jt);
        }
    };
    // tile size of the KB-deep updates and of U: 128 (k_big_wide) with PHIF_WIDE128=1
    const int TW = wide128 ? 128 : T;
    for (int kb0 = 0; kb0 < nmax; kb0 += KB) {
      for (int s0 = kb0; s0 < std::min(nmax, kb0 + KB); s0 += T) {
        Phase ph{0, {0, 0, 0}, {0, 0, 0}, s0, T};
        ph.off[0] = (int64_t)wc.size();
        for (int c = 0; c < nbig; ++c)
          if (n[c] > s0) {
            wc.push_back(c);
            wi.push_back(0);
            wj.push_back(0);
          }
        ph.off[1] = (int64_t)wc.size();
        for (int c = 0; c < nbig; ++c) {
          if (n[c] <= s0) continue;
          const int kb = std::min(T, n[c] - s0), base = s0 + kb;
          const int ntr = (rws[c] - base + T - 1) / T;
          for (int it = 0; it < ntr; ++it) {
            if (zero_tile(c, base + T * it, s0 + kb)) continue;
            wc.push_back(c);
            wi.push_back(it);
            wj.push_back(0);
          }
        }
        ph.off[2] = (int64_t)wc.size();
        for (int c = 0; c < nbig; ++c)
          if (n[c] > s0 + T) trailing(c, s0 + T, std::min(n[c], kb0 + KB), s0 + T);
        ph.cnt[0] = ph.off[1] - ph.off[0];
        ph.cnt[1] = ph.off[2] - ph.off[1];
        ph.cnt[2] = (int64_t)wc.size() - ph.off[2];
        phases.push_back(ph);
      }
      // KB-deep update of the trailing matrix, split for look-ahead: W1 = the next block's
      // columns (stays on the main stream, the next block's steps need it), W2 = the columns
      // beyond the next block (side stream, overlapping the next block's 64-wide chain)
      Phase w1{1, {(int64_t)wc.size(), 0, 0}, {0, 0, 0}, kb0, KB};
      for (int c = 0; c < nbig; ++c)
        if (n[c] > kb0 + KB) trailing(c, kb0 + KB, std::min(n[c], kb0 + 2 * KB), kb0 + KB, TW);
      w1.cnt[0] = (int64_t)wc.size() - w1.off[0];
      if (w1.cnt[0]) phases.push_back(w1);
      Phase w2{3, {(int64_t)wc.size(), 0, 0}, {0, 0, 0}, kb0, KB};
      for (int c = 0; c < nbig; ++c)
        if (n[c] > kb0 + 2 * KB) {
          // tiles of trailing(c, kb0 + KB, n, ..) with column tile index >= KB / T
          const int base = kb0 + KB, kend = kb0 + KB;
          const int nr = (rws[c] - base + TW - 1) / TW, nc = (n[c] - base + TW - 1) / TW;
          for (int it = 0; it < nr; ++it)
            for (int jt = KB / TW; jt < nc; ++jt) {
              if (jt > it && base + TW * (it + 1) <= n[c]) continue;
              if (zero_tile(c, base + TW * it, kend)) continue;
              wc.push_back(c);
              wi.push_back(it);
              wj.push_back(jt);
            }
        }
      w2.cnt[0] = (int64_t)wc.size() - w2.off[0];
      if (w2.cnt[0]) phases.push_back(w2);
    }
    Phase us{2, {(int64_t)wc.size(), 0, 0}, {0, 0, 0}, 0, 0};
    for (int c = 0; c < nbig; ++c) {
      const int nb = (b[c] + TW - 1) / TW;
      for (int it = 0; it < nb; ++it)
        for (int jt = 0; jt <= it; ++jt) {
          wc.push_back(c);
          wi.push_back(it);
          wj.push_back(jt);
        }
    }
    us.cnt[0] = (int64_t)wc.size() - us.off[0];
    if (us.cnt[0]) phases.push_back(us);
    nwork_total = (int64_t)wc.size();
    upload(d_n, n, s);
    upload(d_b, b, s);
    upload(d_rows, rws, s);
    upload(d_op, op, s);
    upload(d_P, Pp, s);
    upload(d_U, Up, s);
    d_linv.alloc((size_t)nbig * T * T * sizeof(double), s);
    upload(d_cell, wc, s);
    upload(d_i, wi, s);
    upload(d_j, wj, s);
  }
  BigArgs args(int64_t off, int64_t cnt, int k0, int kw) const {
    BigArgs a;
    a.ncell = nbig;
    a.n = d_n.as<int>();
    a.b = d_b.as<int>();
    a.rows = d_rows.as<int>();
    a.P = d_P.as<double* const>();
    a.U = d_U.as<double* const>();
    a.Linv = d_linv.as<double>();
    a.op = d_op.as<int>();
    a.w_cell = d_cell.as<int>() + off;
    a.w_i = d_i.as<int>() + off;
    a.w_j = d_j.as<int>() + off;
    a.nwork = (int)cnt;
    a.k0 = k0;
    a.kw = kw;
    return a;
  }
  void run(DevStatus* st, cudaStream_t s) const {
    // Look-ahead: the 64-wide chain (diag, trsm, narrow updates) and W1 (the next block's
    // columns) run on a high-priority stream, W2 (the trailing columns beyond the next block) on
    // the caller's stream; so the chain of block b+1 takes SMs as soon as W2(b)'s CTAs retire
    // instead of queueing behind them. W1(b+1) waits for W2(b) (same C tiles).
    static const bool lookahead = !getenv("PHIF_NO_LOOKAHEAD");
    cudaStream_t hp = lookahead ? prio_stream() : s;
    std::vector<cudaEvent_t> evs;
    auto mark = [&](cudaStream_t from, cudaStream_t to) {   // `to` waits for the work issued on `from`
      if (from == to) return;
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      evs.push_back(e);
      CK(cudaEventRecord(e, from));
      CK(cudaStreamWaitEvent(to, e, 0));
    };
    auto wide = [&](const BigArgs& a, int mode, cudaStream_t st) {
      if (wide128) launch_big_wide(a, mode, st);
      else launch_big_nt(a, mode, st);
    };
    mark(s, hp);
    bool w2_pending = false;
    for (const Phase& ph : phases) {
      if (ph.kind == 0) {
        launch_big_step(args(ph.off[0], ph.cnt[0], ph.k0, ph.kw), args(ph.off[1], ph.cnt[1], ph.k0, ph.kw),
                        args(ph.off[2], ph.cnt[2], ph.k0, ph.kw), st, hp);
      } else if (ph.kind == 3) {
        mark(hp, s);
        wide(args(ph.off[0], ph.cnt[0], ph.k0, ph.kw), 0, s);
        w2_pending = true;
      } else {
        if (w2_pending) mark(s, hp);
        w2_pending = false;
        wide(args(ph.off[0], ph.cnt[0], ph.k0, ph.kw), ph.kind == 1 ? 0 : 1, hp);
      }
    }
    mark(hp, s);
    if (nbig) launch_big_zero_upper(args(0, 0, 0, 0), s);
    for (cudaEvent_t e : evs) cudaEventDestroy(e);   // (destruction is deferred until they complete)
  }
  static cudaStream_t prio_stream() {
    static cudaStream_t st[16] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!st[dev & 15]) {
      int lo = 0, hi = 0;
      CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      CK(cudaStreamCreateWithPriority(&st[dev & 15], cudaStreamNonBlocking, hi));
    }
    return st[dev & 15];
  }
};

}  // namespace

// PHIF_TEAM_PROF=1: accumulate per-phase team CPQR cycles (printed at process exit)
static long long* team_prof_buffer() {
  static long long* buf = nullptr;
  static int on = -1;
  if (on < 0) {
    on = getenv("PHIF_TEAM_PROF") ? 1 : 0;
    if (on) {
      cudaMallocManaged(&buf, 32 * sizeof(long long));
      for (int i = 0; i < 32; ++i) buf[i] = 0;
      atexit([] {
        cudaDeviceSynchronize();
        fprintf(stderr, "[phif] team phases CTA0 (Mcycles): argmax+publish %.1f sync %.1f reflector %.1f pass1(smem) %.1f pass1(L2) %.1f pass2(smem) %.1f pass2(L2) %.1f | steps %lld | QR %.1f [panel %.1f update %.1f syncs %.1f] CPQR %.1f finish %.1f\n",
                buf[0] / 1e6, buf[1] / 1e6, buf[2] / 1e6, buf[3] / 1e6, buf[4] / 1e6, buf[5] / 1e6, buf[6] / 1e6, buf[8], buf[11] / 1e6, buf[14] / 1e6, buf[7] / 1e6, buf[15] / 1e6, buf[12] / 1e6, buf[13] / 1e6);
        fprintf(stderr, "[phif] team QR CTA0: update calls %lld [pass1 %.1f Z %.1f pass2 %.1f Mcycles] factor calls %lld waits %lld\n",
                buf[16], buf[17] / 1e6, buf[18] / 1e6, buf[19] / 1e6, buf[20], buf[21]);
        fprintf(stderr, "[phif] team QR CTA0 factor: load %.1f columns %.1f G/T %.1f store %.1f Mcycles\n", buf[22] / 1e6,
                buf[23] / 1e6, buf[24] / 1e6, buf[25] / 1e6);
        fprintf(stderr, "[phif] team CPQR pass1 CTA0: own-list %.1f chunk-setup %.1f dots %.1f reduce %.1f Mcycles\n",
                buf[26] / 1e6, buf[27] / 1e6, buf[28] / 1e6, buf[29] / 1e6);
      });
    }
  }
  return buf;
}

// PHIF_GID_PROF=1: per-phase clocks of the Gram-path CPQR (CTA 0 of every launch)
static long long* gid_prof_buffer() {
  static long long* buf = nullptr;
  static int on = -1;
  if (on < 0) {
    on = getenv("PHIF_GID_PROF") ? 1 : 0;
    if (on) {
      cudaMallocManaged(&buf, 32 * sizeof(long long));
      for (int i = 0; i < 32; ++i) buf[i] = 0;
      atexit([] {
        cudaDeviceSynchronize();
        fprintf(stderr, "[phif] gid CPQR CTA0 (Mcycles): load %.2f argmax %.2f pieces %.2f barrier %.2f rowread %.2f update %.2f downdate %.2f post %.2f backsub %.2f | steps %lld\n",
                buf[0] / 1e6, buf[1] / 1e6, buf[2] / 1e6, buf[3] / 1e6, buf[4] / 1e6, buf[5] / 1e6, buf[6] / 1e6,
                buf[7] / 1e6, buf[8] / 1e6, buf[9]);
        fprintf(stderr, "[phif] small-separator ID CTA0 (Mcycles): dependency wait %.2f gather-count %.2f copy %.2f gram+cpqr+T %.2f | separators %lld\n",
                buf[19] / 1e6, buf[16] / 1e6, buf[17] / 1e6, buf[18] / 1e6, buf[23]);
        fprintf(stderr, "[phif] banded cell CTA0 (kcycles/cell): load %.1f cholesky %.1f L rows %.1f X %.1f L^-T %.1f U %.1f | cells %lld\n",
                buf[24] / 1e3 / std::max(1LL, buf[30]), buf[25] / 1e3 / std::max(1LL, buf[30]), buf[26] / 1e3 / std::max(1LL, buf[30]),
                buf[27] / 1e3 / std::max(1LL, buf[30]), buf[28] / 1e3 / std::max(1LL, buf[30]), buf[29] / 1e3 / std::max(1LL, buf[30]), buf[30]);
      });
    }
  }
  return buf;
}

// Pinned staging ring for host -> device uploads: two halves; every copy issued from a half
// records its own event (on whichever stream issued it), and a half is refilled only after all
// of its copies have drained. The host fills the staging area with a parallel memcpy, so the DMA
// engine copies at pinned-memory speed instead of the driver's pageable staging.
void upload_bytes(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  static constexpr size_t HALF = (size_t)96 << 20, MIN_STAGED = (size_t)1 << 20;
  static char* ring = nullptr;
  static bool ok = true;
  static std::vector<cudaEvent_t> pending[2], spare;
  static int cur = 0;
  static size_t pos = 0;
  static std::mutex mu;
  if (bytes < MIN_STAGED || !ok) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    return;
  }
  std::lock_guard<std::mutex> lock(mu);
  if (!ring) {
    if (cudaHostAlloc((void**)&ring, 2 * HALF, cudaHostAllocDefault) != cudaSuccess) {
      cudaGetLastError();
      ok = false;
      CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
      return;
    }
  }
  const char* sp = static_cast<const char*>(src);
  char* dp = static_cast<char*>(dst);
  while (bytes > 0) {
    if (pos == HALF) {   // switch halves; wait until every copy from the other half has drained
      cur ^= 1;
      pos = 0;
      for (cudaEvent_t e : pending[cur]) {
        CK(cudaEventSynchronize(e));
        spare.push_back(e);
      }
      pending[cur].clear();
    }
    const size_t len = std::min(bytes, HALF - pos);
    char* stage = ring + (size_t)cur * HALF + pos;
    const int64_t nchunk = (int64_t)std::max<size_t>(1, len >> 20);
    // a few threads saturate the host memory bandwidth; the rest of the cores stay free for the
    // planner's helper threads (a statically scheduled team waiting on a preempted thread stalls)
#pragma omp parallel for schedule(dynamic, 1) num_threads(std::min<int64_t>(nchunk, 6))
    for (int64_t c = 0; c < nchunk; ++c) {
      const size_t a = len * c / nchunk, e = len * (c + 1) / nchunk;
      memcpy(stage + a, sp + a, e - a);
    }
    CK(cudaMemcpyAsync(dp, stage, len, cudaMemcpyHostToDevice, s));
    cudaEvent_t e;
    if (spare.empty()) {
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    } else {
      e = spare.back();
      spare.pop_back();
    }
    CK(cudaEventRecord(e, s));
    pending[cur].push_back(e);
    pos += len;
    sp += len;
    dp += len;
    bytes -= len;
  }
}

// device -> host copy through a pinned staging buffer (DMA into pinned memory, then a parallel
// host memcpy out); synchronises the stream
void download_bytes(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  static constexpr size_t CH = (size_t)16 << 20;   // (small: pinning the staging area is paid by the first call)
  static char* stage = nullptr;
  static bool ok = true;
  static std::mutex mu;
  if (bytes < ((size_t)1 << 20) || !ok) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return;
  }
  std::lock_guard<std::mutex> lock(mu);
  if (!stage && cudaHostAlloc((void**)&stage, 2 * CH, cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    ok = false;
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return;
  }
  // double-buffered: the DMA of chunk c+1 overlaps the host copy of chunk c
  const size_t nch = (bytes + CH - 1) / CH;
  cudaEvent_t ev[2];
  CK(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  auto issue = [&](size_t c) {
    const size_t a = c * CH, len = std::min(CH, bytes - a);
    CK(cudaMemcpyAsync(stage + (c & 1) * CH, static_cast<const char*>(src) + a, len, cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(ev[c & 1], s));
  };
  issue(0);
  for (size_t c = 0; c < nch; ++c) {
    if (c + 1 < nch) issue(c + 1);
    CK(cudaEventSynchronize(ev[c & 1]));
    const size_t a = c * CH, len = std::min(CH, bytes - a);
    const char* from = stage + (c & 1) * CH;
    char* to = static_cast<char*>(dst) + a;
    const int64_t np = (int64_t)std::max<size_t>(1, len >> 21);
#pragma omp parallel for schedule(dynamic, 1) num_threads(std::min<int64_t>(np, 6))
    for (int64_t q = 0; q < np; ++q) {
      const size_t u = len * q / np, e = len * (q + 1) / np;
      memcpy(to + u, from + u, e - u);
    }
  }
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
}

static void keep_pool_memory() {
  // freed blocks stay in the stream-ordered pool instead of going back to the driver at every sync
  static bool done = false;
  if (done) return;
  done = true;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
}

std::unique_ptr<Factorization> factorize(const Matrix& A, int dim, int n, int m, double eps, int method,
                                         cudaStream_t s, bool timing) {
  configure_kernels();
  keep_pool_memory();
  // the planner's OpenMP teams leave two cores to the helper threads (boundary reduction lists,
  // staging copies): a statically scheduled team waiting on a preempted thread stalls
  static const int omp_once = [] {
    // main team + pre-plan team + the reduction-list helper stay within the host's cores
    if (!getenv("OMP_NUM_THREADS"))
      omp_set_num_threads(std::max(1, omp_get_num_procs() - std::max(2, omp_get_num_procs() / 4) - 2));
    return 0;
  }();
  (void)omp_once;
  g_dbg_t0 = std::chrono::steady_clock::now();
  auto F = std::make_unique<Factorization>();
  F->spec.init(dim, n, m);
  F->method = method;
  F->eps = method == 2 ? 0.0 : eps;
  F->stream = s;
  const Spec& sp = F->spec;
  if (sp.N != A.N) throw std::runtime_error("matrix order does not match the grid spec");
  auto t_start = clk::now();
  double plan_ms = 0.0;
  F->alive.alloc(sp.N * sizeof(int), s);
  launch_fill_int(F->alive.as<int>(), 1, sp.N, s);
  DBG("alive initialised");
  F->status.alloc(sizeof(DevStatus), s);
  cudaEvent_t ev[16];
  if (timing)
    for (auto& e : ev) CK(cudaEventCreate(&e));

  std::vector<std::pair<int, int>> pairs;
  std::vector<uint8_t> alive_mem;  // survivors of the previous level, per member position
  std::future<LevelPlan> preplan;  // structure of the next level, planned while the IDs run
  // the pre-plan completed with the survivors (sizes, offsets), on a host thread while the GPU
  // runs the skeleton updates
  std::future<std::pair<LevelPlan, bool>> fin_task;
  static const bool no_preplan = getenv("PHIF_NO_PREPLAN") != nullptr;
  try {
  for (int lev = 0; lev <= sp.L; ++lev) {
    auto tp = clk::now();
    const auto t_level0 = tp;
    F->levels.push_back(std::make_unique<LevelRT>());
    LevelRT& L = *F->levels.back();
    LevelRT* prev = lev > 0 ? F->levels[lev - 1].get() : nullptr;
    // level 0 is planned on the device when its cells take the one-CTA path (gpu_plan.cu;
    // PHIF_HOST_PLAN=1 forces the host planner)
    static const bool host_plan = getenv("PHIF_HOST_PLAN") != nullptr;
    DevPlan0 dp;
    if (lev == 0 && !host_plan && gpu_plan0_applicable(sp, BIG_CELL)) {
      plan_level0_device(sp, A.rowptr.as<int64_t>(), A.col.as<int>(), A.nnz, L.plan, dp, s);
      DBG("level 0: planned on the device G=%d blocks=%lld", L.plan.grp.G, (long long)dp.nblocks);
    } else {
      bool done = false;
      if (lev > 0 && fin_task.valid()) {
        auto res = fin_task.get();
        if (res.second) {
          L.plan = std::move(res.first);
          done = true;
          DBG("level %d: pre-plan finished G=%d", lev, L.plan.grp.G);
        }
      }
      if (!done) {
      if (lev == 0) {
        A.ensure_host_pattern(s);
        L.plan.grp = classify_all(sp);
        DBG("level 0: classified");
        pairs = pattern_from_csr(L.plan.grp, sp.N, A.h_rowptr.get(), A.h_col.get());
      } else {
        L.plan.grp = classify_next(sp, prev->plan.grp, alive_mem);
        pairs = pattern_next(prev->plan, L.plan.grp);
      }
      DBG("level %d: grouped G=%d", lev, L.plan.grp.G);
      build_level(sp, L.plan, std::move(pairs));
      }
    }
    // the next level's structure only depends on this level's plan: it is planned on a host
    // thread while this level's host descriptors are built and its kernels run
    if (!L.plan.root && !no_preplan)
      preplan = std::async(std::launch::async, [&sp, &L]() {
        omp_set_num_threads(std::max(2, omp_get_num_procs() / 4));   // (small team; see below)
        return preplan_next(sp, L.plan);
      });
    // device copy of a plan array: taken over from the device planner, else uploaded
    auto dev_arr = [&](DBuf& dst, DBuf& from, const auto& host) {
      if (dp.valid) dst = std::move(from);
      else upload(dst, host, s);
    };
    DBG("level %d: planned blocks=%zu pool=%lld", lev, L.plan.pat.bg.size(), (long long)L.plan.pool_doubles);
    const LevelPlan& P = L.plan;
    const Groups& G = P.grp;
    L.S = (int64_t)G.mem.size();
    // ---------------- host-side descriptors for this level ----------------
    const int p = (int)P.interior.size();
    std::vector<int64_t> P_off(p), U_off(p), I_off(p), B_off(p), cwork(p);
    std::vector<int> nbr_w(P.cell_nbr.size());
    auto Bdofs_p = std::make_shared<std::vector<int>>();   // shared with the reduction-list task
    std::vector<int>& Bdofs = *Bdofs_p;
    int64_t rec = 0, uacc = 0, bacc = 0, wacc = 0;
    for (int t = 0; t < p; ++t) {
      const int nn = P.cell_n[t], bb = P.cell_b[t];
      P_off[t] = rec;
      rec += (int64_t)(nn + bb) * nn;
      rec += (int64_t)nn * nn;   // identity rows -> L^-T for the GEMM replay
      U_off[t] = uacc;
      uacc += (int64_t)bb * bb;
      I_off[t] = G.off[P.interior[t]];
      B_off[t] = bacc;
      bacc += bb;
      cwork[t] = wacc;
      wacc += 2 * nn + bb;
    }
    // boundary DOFs of every cell (cell order, neighbour order, members ascending), in parallel
    Bdofs.resize(bacc);
#pragma omp parallel for schedule(dynamic, 256)
    for (int t = 0; t < p; ++t) {
      int64_t o = B_off[t];
      for (int64_t j = P.cell_nbr_off[t]; j < P.cell_nbr_off[t + 1]; ++j) {
        const int h = P.cell_nbr[j];
        nbr_w[j] = G.size(h);
        for (int64_t q = G.off[h]; q < G.off[h + 1]; ++q) Bdofs[o++] = G.mem[q];
      }
    }
    L.cell_work_unit = wacc;
    L.wbuf_unit = bacc;
    for (int t = 0; t < p; ++t) {
      L.cell_nmax = std::max(L.cell_nmax, P.cell_n[t]);
      L.cell_bmax = std::max(L.cell_bmax, P.cell_b[t]);
    }
    DBG("level %d: host: cell descriptors", lev);
    {
      double f1 = 0.0, b1 = 0.0, b0 = 0.0;
#pragma omp parallel for reduction(+ : f1, b1)
      for (int t = 0; t < p; ++t) {
        const double nn = P.cell_n[t], bb = P.cell_b[t];
        f1 += nn * nn * nn / 3.0 + nn * nn * bb + nn * bb * bb;
        b1 += 8.0 * (nn * nn + nn * bb + (nn + bb) * nn + bb * bb);
      }
      const int64_t ntgt = (int64_t)P.tgt_blk.size(), nblkp = (int64_t)P.pat.bg.size();
#pragma omp parallel for reduction(+ : b1)
      for (int64_t q = 0; q < ntgt; ++q) {
        const int blk = P.tgt_blk[q];
        b1 += 8.0 * 2.0 * G.size(P.pat.bg[blk]) * G.size(P.pat.bh[blk]);
      }
#pragma omp parallel for reduction(+ : b0)
      for (int64_t b = 0; b < nblkp; ++b) b0 += 8.0 * 2.0 * G.size(P.pat.bg[b]) * G.size(P.pat.bh[b]);
      L.fl[1] += f1;
      L.by[1] += b1;
      L.by[0] += b0;
    }
    DBG("level %d: host: boundary reduction lists", lev);
    // record sizes of the block-Jacobi groups and separators (their offsets are formed later,
    // while the GPU eliminates the cells): the pool is allocated for the total now
    const int r = P.root ? 0 : (int)P.precond.size();
    const bool do_prec = (method != 0) && !P.root;
    const int nsk = P.root ? 0 : (int)P.skeleton.size();
    int64_t rec_prec = 0, rec_skel = 0;
#pragma omp parallel for reduction(+ : rec_prec)
    for (int t = 0; t < r; ++t) {
      const int64_t k = G.size(P.precond[t]);
      rec_prec += do_prec ? 2 * k * k : 0;
    }
#pragma omp parallel for reduction(+ : rec_skel)
    for (int t = 0; t < nsk; ++t) {
      const int64_t k = G.size(P.skeleton[t]);
      rec_skel += 3 * k * k;
    }
    const int64_t rec_total = rec + rec_prec + rec_skel;
    L.rec_doubles = rec_total;
    plan_ms += ms_since(tp);
    L.t_ms[5] += ms_since(tp);
    // boundary reduction lists (x_B -= X^T y in fixed cell order): only the apply needs them,
    // so they are built on a host thread (started after the OpenMP planning loops) while the GPU
    // factors, and uploaded after the level loop
    L.bd_task = std::async(std::launch::async, [Bdp = std::shared_ptr<const std::vector<int>>(Bdofs_p)]() {
      const std::vector<int>& Bd = *Bdp;
      // rows of every boundary DOF in cell order: counting sort over the DOF range
      BdLists out;
      if (Bd.empty()) {
        out.off.push_back(0);
        return out;
      }
      const auto mm = std::minmax_element(Bd.begin(), Bd.end());
      const int lo = *mm.first, span = *mm.second - lo + 1;
      std::vector<int64_t> start(span + 1, 0);
      for (int d : Bd) start[d - lo + 1]++;
      for (int d = 0; d < span; ++d) {
        if (start[d + 1]) {
          out.dof.push_back(d + lo);
          out.off.push_back(start[d]);
        }
        start[d + 1] += start[d];
      }
      out.off.push_back((int64_t)Bd.size());
      out.rows.resize(Bd.size());
      for (size_t i = 0; i < Bd.size(); ++i) out.rows[start[Bd[i] - lo]++] = (int)i;
      return out;
    });
    // ---------------- device structures ----------------
    DBG("level %d: rec=%lld", lev, (long long)rec);
    if (dp.valid) {
      L.goff = std::move(dp.goff);
      L.mem = std::move(dp.mem);
      L.gsize = std::move(dp.gsize);
      L.boff = std::move(dp.boff);
      L.bg = std::move(dp.bg);
      L.bh = std::move(dp.bh);
      L.adj_off = std::move(dp.adj_off);
      L.adj_nbr = std::move(dp.adj_nbr);
      L.adj_blk = std::move(dp.adj_blk);
      L.diag_blk = std::move(dp.diag_blk);
    } else {
      upload_structure(L, s);
    }
    DBG("level %d: structure uploaded", lev);
    L.pool.alloc(std::max<int64_t>(P.pool_doubles, 1) * sizeof(double), s, /*zero=*/true);
    if (debug_on()) cudaStreamSynchronize(s);
    DBG("level %d: pool allocated", lev);
    L.rec.alloc(std::max<int64_t>(rec_total, 1) * sizeof(double), s);
    if (debug_on()) cudaStreamSynchronize(s);
    DBG("level %d: records allocated", lev);
    F->rec_bytes += rec_total * (int64_t)sizeof(double);
    LevelDev dv = L.dev();
    int band_w = 0, band_nmax = 0, band_bmax = 0;   // banded level-0 cells (2D), set below
    if (timing) CK(cudaEventRecord(ev[0], s));
    if (lev == 0) {
      DBuf dgid, dpos;
      dgid.alloc(sp.N * sizeof(int), s);
      dpos.alloc(sp.N * sizeof(int), s);
      launch_group_pos(dv, dgid.as<int>(), dpos.as<int>(), s);
      launch_ingest(dv, dgid.as<int>(), dpos.as<int>(), A.rowptr.as<int64_t>(), A.col.as<int>(),
                    A.val.as<double>(), sp.N, s);
      // 2D level-0 cells too big for the one-CTA kernel: banded path when every interior group's
      // couplings stay within w = m-1 positions (natural order; checked on the device)
      static const bool no_band = getenv("PHIF_NO_BAND") != nullptr;
      int nmax = 0, bmax = 0;
      for (int t = 0; t < p; ++t) {
        nmax = std::max(nmax, P.cell_n[t]);
        bmax = std::max(bmax, P.cell_b[t]);
      }
      if (!no_band && sp.dim == 2 && nmax >= BIG_CELL && band_cells_fit(nmax, bmax, sp.m - 1)) {
        std::vector<uint8_t> isint(G.G);
        for (int gi = 0; gi < G.G; ++gi) isint[gi] = G.kind[gi] == 0;
        DBuf dint, dflag;
        upload(dint, isint, s);
        dflag.alloc(sizeof(int), s, true);
        launch_band_check(A.rowptr.as<int64_t>(), A.col.as<int>(), dgid.as<int>(), dpos.as<int>(),
                          dint.as<uint8_t>(), sp.N, sp.m - 1, dflag.as<int>(), s);
        int flag = 1;
        CK(cudaMemcpyAsync(&flag, dflag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        band_w = flag ? 0 : sp.m - 1;
        band_nmax = nmax;
        band_bmax = bmax;
      }
      // (stream-ordered: no host sync needed here; buffers are recycled on the same stream)
    } else {
      RepackArgs ra;
      ra.nblk = (int)P.pat.bg.size();
      ra.nbg = L.bg.as<int>();
      ra.nbh = L.bh.as<int>();
      ra.nboff = L.boff.as<int64_t>();
      ra.ngoff = L.goff.as<int64_t>();
      DBuf sg, spos, sloc, slo, sl, wb, wr, wn;
      upload(sg, G.src_group, s);
      upload(spos, G.src_pos, s);
      upload(sloc, G.src_local, s);
      upload(slo, G.srcl_off, s);
      upload(sl, G.srcl, s);
      ra.nsrc_group = sg.as<int>();
      ra.nsrc_pos = spos.as<int>();
      ra.nsrc_local = sloc.as<int>();
      ra.nsrcl_off = slo.as<int64_t>();
      ra.nsrcl = sl.as<int>();
      {
        // row chunks of ~8K elements (at least one row per warp)
        std::vector<int> wbh, wrh, wnh;
        int cap = 1;
        for (size_t b = 0; b < P.pat.bg.size(); ++b) {
          const int gg = P.pat.bg[b], hh = P.pat.bh[b];
          const int rows = G.size(gg), cols = G.size(hh);
          cap = std::max<int>(cap, (int)((G.srcl_off[gg + 1] - G.srcl_off[gg]) * (G.srcl_off[hh + 1] - G.srcl_off[hh])));
          const int step = std::max(8, 8192 / std::max(cols, 1));
          for (int r0 = 0; r0 < rows; r0 += step) {
            wbh.push_back((int)b);
            wrh.push_back(r0);
            wnh.push_back(std::min(step, rows - r0));
          }
        }
        upload(wb, wbh, s);
        upload(wr, wrh, s);
        upload(wn, wnh, s);
        if (cap > 12000) throw std::runtime_error("repack: too many source groups per block pair");
        ra.nwork = (int)wbh.size();
        ra.tab_cap = cap;
        ra.w_blk = wb.as<int>();
        ra.w_row0 = wr.as<int>();
        ra.w_nrow = wn.as<int>();
      }
      ra.npool = L.pool.as<double>();
      ra.opool = prev->pool.as<double>();
      ra.oboff = prev->boff.as<int64_t>();
      ra.oadj_off = prev->adj_off.as<int64_t>();
      ra.oadj_nbr = prev->adj_nbr.as<int>();
      ra.oadj_blk = prev->adj_blk.as<int>();
      ra.ogsize = prev->gsize.as<int>();
      launch_repack(ra, s);
      // (stream-ordered: no host sync needed here; buffers are recycled on the same stream)
      prev->pool.release();
    }
    if (timing) CK(cudaEventRecord(ev[1], s));
    DBG("level %d: ingest/repack done", lev);
    // ---------------- stage 1: cell elimination ----------------
    dev_arr(L.c_interior, dp.interior, P.interior);
    dev_arr(L.c_nbr_off, dp.cell_nbr_off, P.cell_nbr_off);
    dev_arr(L.c_nbr_blk, dp.cell_nbr_blk, P.cell_nbr_blk);
    dev_arr(L.c_nbr_col, dp.cell_nbr_col, P.cell_nbr_col);
    dev_arr(L.c_nbr_w, dp.cell_nbr_w, nbr_w);
    dev_arr(L.c_n, dp.cell_n, P.cell_n);
    dev_arr(L.c_b, dp.cell_b, P.cell_b);
    upload(L.c_P_off, P_off, s);
    upload(L.c_U_off, U_off, s);
    upload(L.c_I_off, I_off, s);
    upload(L.c_B, Bdofs, s);
    upload(L.c_B_off, B_off, s);
    upload(L.c_work_off, cwork, s);
    DBuf U;
    U.alloc(std::max<int64_t>(uacc, 1) * sizeof(double), s);
    CellArgs ca;
    ca.p = p;
    ca.interior = L.c_interior.as<int>();
    ca.nbr_off = L.c_nbr_off.as<int64_t>();
    ca.nbr_blk = L.c_nbr_blk.as<int>();
    ca.nbr_col = L.c_nbr_col.as<int>();
    ca.nbr_w = L.c_nbr_w.as<int>();
    ca.n = L.c_n.as<int>();
    ca.b = L.c_b.as<int>();
    ca.rec = L.rec.as<double>();
    ca.P_off = L.c_P_off.as<int64_t>();
    ca.U = U.as<double>();
    ca.U_off = L.c_U_off.as<int64_t>();
    ca.list = nullptr;
    CK(cudaMemsetAsync(F->status.p, 0xff, sizeof(DevStatus), s));
    // small cells: one CTA each; big cells (n >= BIG_N): tile-parallel 64-wide steps
    std::vector<int> small_cells, big_cells;
    for (int t = 0; t < p; ++t) (P.cell_n[t] >= BIG_CELL ? big_cells : small_cells).push_back(t);
    DBG("level %d: cells p=%d (big %zu)", lev, p, big_cells.size());
    upload(L.d_small_cells, small_cells, s);
    L.h_small_cells = small_cells;
    L.h_big_cells = big_cells;
    L.h_P_off = P_off;
    L.h_I_off = I_off;
    L.h_B_off = B_off;
    L.h_cwork = cwork;
    BigPlan bp;
    const bool banded = band_w > 0 && !big_cells.empty();
    if (banded) {   // algorithmic work of the banded cells: POTRF n w^2, TRSM 2 n w b, SYRK n b^2
      double fd = 0.0, fb = 0.0;
      for (int t : big_cells) {
        const double nn = P.cell_n[t], bb = P.cell_b[t], ww = band_w;
        fd += nn * nn * nn / 3.0 + nn * nn * bb + nn * bb * bb;
        fb += nn * ww * ww + 2.0 * nn * ww * bb + nn * bb * bb;
      }
      L.fl[1] += fb - fd;
    }
    if (!big_cells.empty() && !banded)
      bp.build(big_cells, P.cell_n, P.cell_b, L.rec.as<double>(), P_off, U.as<double>(), U_off, s);
    DBG("level %d: big plan built (%lld work items)", lev, (long long)bp.nwork_total);
    if (!big_cells.empty()) upload(bp.d_list, big_cells, s);
    if (timing) CK(cudaEventRecord(ev[2], s));
    if (!small_cells.empty()) {
      ca.list = L.d_small_cells.as<int>();
      launch_cell(dv, ca, (int)small_cells.size(), F->status.as<DevStatus>(), s);
    }
    if (banded) {
      DBuf scratch;   // band of L + reciprocals per cell, from the one-warp Cholesky
      scratch.alloc((size_t)big_cells.size() * band_scratch_stride(band_nmax, band_w) * sizeof(double), s);
      launch_cell_band(dv, ca, bp.d_list.as<int>(), (int)big_cells.size(), band_nmax, band_bmax, band_w,
                       scratch.as<double>(), F->status.as<DevStatus>(), gid_prof_buffer(), s);
    } else if (!big_cells.empty()) {
      launch_big_build(dv, ca, bp.d_list.as<int>(), (int)big_cells.size(), s);
      bp.run(F->status.as<DevStatus>(), s);
    }
    if (timing) CK(cudaEventRecord(ev[3], s));
    // (below the root the cell-stage status is read after the block-Jacobi descriptors are built,
    // so that host work overlaps the elimination; nothing reads the factor before that check)
    if (P.root) check_status(*F, lev, ST_ROOT);
    DBG("level %d: cells done", lev);
    DBuf tb, to, cc, cr, ccol;
    dev_arr(tb, dp.tgt_blk, P.tgt_blk);
    dev_arr(to, dp.tgt_off, P.tgt_off);
    dev_arr(cc, dp.con_cell, P.con_cell);
    dev_arr(cr, dp.con_row, P.con_row);
    dev_arr(ccol, dp.con_col, P.con_col);
    SchurArgs sa;
    sa.ntgt = (int)P.tgt_blk.size();
    sa.tgt_blk = tb.as<int>();
    sa.tgt_off = to.as<int64_t>();
    sa.con_cell = cc.as<int>();
    sa.con_row = cr.as<int>();
    sa.con_col = ccol.as<int>();
    sa.cell_b = L.c_b.as<int>();
    sa.U = U.as<double>();
    sa.U_off = L.c_U_off.as<int64_t>();
    if (timing) CK(cudaEventRecord(ev[4], s));
    DBG("level %d: schur targets=%d", lev, sa.ntgt);
    launch_schur(dv, sa, s);
    if (timing) CK(cudaEventRecord(ev[5], s));
    U.release();
    if (P.root) {
      if (timing) {
        CK(cudaEventSynchronize(ev[5]));
        float a;
        cudaEventElapsedTime(&a, ev[0], ev[1]); L.t_ms[0] = a;
        cudaEventElapsedTime(&a, ev[2], ev[3]); L.t_ms[1] = a;
        cudaEventElapsedTime(&a, ev[4], ev[5]); L.t_ms[1] += a;
      }
      L.pool.release();
      break;
    }
    // ---------------- stage 2: block Jacobi ----------------
    auto t_ov = clk::now();   // (host work overlapped with the GPU's cell elimination)
    // precondition records
    std::vector<int64_t> L_off(r), Lg_off(G.G, -1), pI_off(r), pwork(r);
    std::vector<int> pn(r);
    int64_t pw = 0;
    for (int t = 0; t < r; ++t) {
      const int g = P.precond[t], k = G.size(g);
      if (do_prec) {
        L_off[t] = rec;
        Lg_off[g] = rec;
        rec += 2 * (int64_t)k * k;   // [L ; L^-T]
      }
      pn[t] = k;
      pI_off[t] = G.off[g];
      pwork[t] = pw;
      pw += (k >= APPLY_BIG ? 2 : 1) * k;
    }
    L.prec_work_unit = pw;
    L.h_L_off = L_off;
    L.h_pI_off = pI_off;
    L.h_pwork = pwork;
    L.h_pn = pn;
    if (do_prec) {
      double f2 = 0.0, b2 = 0.0;
#pragma omp parallel for reduction(+ : f2, b2)
      for (int t = 0; t < r; ++t) {
        const double k = pn[t];
        f2 += k * k * k / 3.0;
        b2 += 8.0 * 3.0 * k * k;
      }
      const int64_t nsc = (int64_t)P.scale_blk.size();
#pragma omp parallel for reduction(+ : f2, b2)
      for (int64_t q = 0; q < nsc; ++q) {
        const int b = P.scale_blk[q];
        const double kg = G.size(P.pat.bg[b]), kh = G.size(P.pat.bh[b]);
        f2 += kg * kg * kh + kg * kh * kh;
        b2 += 8.0 * 2.0 * kg * kh;
      }
      L.fl[2] += f2;
      L.by[2] += b2;
    }
    DBG("level %d: host: precondition records", lev);
    L.t_host_overlap_ms += ms_since(t_ov);
    check_status(*F, lev, ST_ELIMINATE);
    dev_arr(L.p_groups, dp.precond, P.precond);
    upload(L.p_L_off, L_off, s);
    upload(L.p_L_off_of_group, Lg_off, s);
    dev_arr(L.p_scale_blk, dp.scale_blk, P.scale_blk);
    upload(L.p_n, pn, s);
    upload(L.p_I_off, pI_off, s);
    upload(L.p_work_off, pwork, s);
    PrecArgs pa;
    pa.r = do_prec ? r : 0;
    pa.groups = L.p_groups.as<int>();
    pa.rec = L.rec.as<double>();
    pa.L_off = L.p_L_off.as<int64_t>();
    pa.L_off_of_group = L.p_L_off_of_group.as<int64_t>();
    pa.nscale = do_prec ? (int)P.scale_blk.size() : 0;
    pa.scale_blk = L.p_scale_blk.as<int>();
    pa.list = nullptr;
    pa.scale_list = nullptr;
    if (timing) CK(cudaEventRecord(ev[6], s));
    DBG("level %d: precondition r=%d scale=%d", lev, pa.r, pa.nscale);
    if (do_prec) {
      // small groups: one CTA each; big groups: tile-parallel panels [A_gg ; I] -> [L ; L^-T]
      std::vector<int> ptiny, psmall, pbig;
      int tiny_max = 1;
      const int kmax_pr = r ? *std::max_element(pn.begin(), pn.end()) : 1;
      const bool all_tiny = kmax_pr <= 32;   // (level 0: no host lists, the warp kernels take all)
      if (all_tiny) tiny_max = std::max(1, kmax_pr);
      for (int t = 0; t < r && !all_tiny; ++t) {
        if (pn[t] <= 32) {
          ptiny.push_back(t);
          tiny_max = std::max(tiny_max, pn[t]);
        } else {
          (pn[t] >= BIG_PREC ? pbig : psmall).push_back(t);
        }
      }
      L.h_prec_big = pbig;
      upload(L.d_prec_small, psmall, s);
      PrecArgs ps = pa;
      ps.list = L.d_prec_small.as<int>();
      ps.r = (int)psmall.size();
      launch_prec_factor(dv, ps, F->status.as<DevStatus>(), s);
      DBuf dtiny;
      if (!all_tiny) upload(dtiny, ptiny, s);
      launch_prec_factor_warp(dv, pa, all_tiny ? nullptr : dtiny.as<int>(), all_tiny ? r : (int)ptiny.size(), tiny_max,
                              F->status.as<DevStatus>(), s);
      if (!pbig.empty()) {
        DBuf dbig;
        upload(dbig, pbig, s);
        launch_prec_build(dv, pa, dbig.as<int>(), (int)pbig.size(), s);
        std::vector<int> zeros(r, 0);
        std::vector<int64_t> zoff(r, 0);
        BigPlan bpp;
        bpp.build(pbig, pn, zeros, L.rec.as<double>(), L_off, L.rec.as<double>(), zoff, s);
        bpp.run(F->status.as<DevStatus>(), s);
      }
      DBG("level %d: precondition factor launched", lev);   // (status read before the IDs)
      // two-sided scaling: small blocks by substitution, blocks touching a big group by GEMMs
      // with the explicit inverses: B <- (L_g^-T)^T B L_h^-T
      std::vector<int> stiny, ssmall;
      std::vector<GemmDesc> d1, d2;
      std::vector<int> w1d, w1t, w2d, w2t;
      int64_t tmp_need = 0;
      int stiny_max = 1;
      bool ssmall_gemm = true;   // every mid-size block fits the two-GEMM kernel
      if (all_tiny) stiny_max = tiny_max;   // (every scaled block couples two tiny groups)
      for (size_t q = 0; q < P.scale_blk.size() && !all_tiny; ++q) {
        const int b = P.scale_blk[q];
        const int kg = G.size(P.pat.bg[b]), kh = G.size(P.pat.bh[b]);
        if (std::max(kg, kh) <= 32) {
          stiny.push_back((int)q);
          stiny_max = std::max(stiny_max, std::max(kg, kh));
        } else if (std::max(kg, kh) < BIG_PREC) {
          ssmall.push_back((int)q);
          ssmall_gemm = ssmall_gemm && kg * kh <= 64 * 64;
        } else {
          tmp_need += (int64_t)kg * kh;
        }
      }
      upload(L.d_scale_small, ssmall, s);
      PrecArgs pss = pa;
      pss.scale_list = L.d_scale_small.as<int>();
      pss.nscale = (int)ssmall.size();
      launch_prec_scale(dv, pss, s, ssmall_gemm);
      DBuf dstiny;
      if (!all_tiny) upload(dstiny, stiny, s);
      launch_prec_scale_warp(dv, pa, all_tiny ? nullptr : dstiny.as<int>(),
                             all_tiny ? (int)P.scale_blk.size() : (int)stiny.size(), stiny_max, s);
      if (tmp_need) {
        DBuf tmp;
        tmp.alloc(tmp_need * sizeof(double), s);
        int64_t to = 0;
        const double* rec0 = L.rec.as<double>();
        for (size_t q = 0; q < P.scale_blk.size(); ++q) {
          const int b = P.scale_blk[q];
          const int gg = P.pat.bg[b], hh = P.pat.bh[b];
          const int kg = G.size(gg), kh = G.size(hh);
          if (std::max(kg, kh) < BIG_PREC) continue;
          double* blk = L.pool.as<double>() + P.boff[b];
          double* T = tmp.as<double>() + to;
          to += (int64_t)kg * kh;
          // L_g^-1 (op of the stored L_g^-T) is lower triangular, L_h^-T upper triangular
          GemmDesc a{rec0 + Lg_off[gg] + (int64_t)kg * kg, blk, T, kg, kh, kg, kg, kh, kh, 1, 1.0, 0.0, 1};
          GemmDesc c{T, rec0 + Lg_off[hh] + (int64_t)kh * kh, blk, kg, kh, kh, kh, kh, kh, 0, 1.0, 0.0, 2};
          for (int t = 0; t < (kg + 63) / 64; ++t) {
            w1d.push_back((int)d1.size());
            w1t.push_back(t);
            w2d.push_back((int)d2.size());
            w2t.push_back(t);
          }
          d1.push_back(a);
          d2.push_back(c);
        }
        DBuf dd1, dd2, dw1d, dw1t, dw2d, dw2t;
        upload(dd1, d1, s);
        upload(dd2, d2, s);
        upload(dw1d, w1d, s);
        upload(dw1t, w1t, s);
        upload(dw2d, w2d, s);
        upload(dw2t, w2t, s);
        launch_bgemm(dd1.as<GemmDesc>(), dw1d.as<int>(), dw1t.as<int>(), (int)w1d.size(), s);
        launch_bgemm(dd2.as<GemmDesc>(), dw2d.as<int>(), dw2t.as<int>(), (int)w2d.size(), s);
        // (stream-ordered: no host sync needed here; buffers are recycled on the same stream)
      }
    }
    if (timing) CK(cudaEventRecord(ev[7], s));
    // ---------------- stage 3: skeletonization ----------------
    t_ov = clk::now();   // (overlapped with the block-Jacobi stage)
    if (nsk && L.plan.wave_order.empty()) compute_waves(L.plan, G.G);   // (device-planned level 0)
    // skeleton records / workspaces (upper bounds; ranks known after the ID)
    std::vector<int64_t> T_off(nsk), SP_off(nsk), work_off(nsk), iwork_off(nsk), awork(nsk), rows_bound(nsk);
    int64_t work = 0, iwork = 0, aw = 0;
#pragma omp parallel for schedule(static)
    for (int t = 0; t < nsk; ++t) {   // coupled rows per separator (the prefix sums follow)
      int64_t rows = 0;
      for (int64_t q = P.sk_nbr_off[t]; q < P.sk_nbr_off[t + 1]; ++q) rows += G.size(P.sk_nbr[q]);
      rows_bound[t] = rows;
    }
    for (int t = 0; t < nsk; ++t) {
      const int g = P.skeleton[t], k = G.size(g);
      const int64_t rows = rows_bound[t];
      T_off[t] = rec;
      rec += (int64_t)k * k;
      SP_off[t] = rec;
      rec += 2 * (int64_t)k * k;   // [L~ ; X~^T ; L~^-T]
      work_off[t] = work;
      work += std::max<int64_t>((std::max<int64_t>(rows, 1)) * k + 2 * k, 2 * (int64_t)k * k);
      iwork_off[t] = iwork;
      iwork += 3 * (int64_t)k;
      awork[t] = aw;
      aw += (k >= APPLY_BIG ? 2 : 1) * k;
    }
    L.skel_work_unit = aw;
    L.h_T_off = T_off;
    L.h_SP_off = SP_off;
    L.h_awork = awork;
    if (rec != rec_total) throw std::runtime_error("record pool layout mismatch");
    L.t_host_overlap_ms += ms_since(t_ov);
    if (do_prec) check_status(*F, lev, ST_PRECONDITION);
    dev_arr(L.s_groups, dp.skeleton, P.skeleton);
    dev_arr(L.s_nbr_off, dp.sk_nbr_off, P.sk_nbr_off);
    dev_arr(L.s_nbr, dp.sk_nbr, P.sk_nbr);
    dev_arr(L.s_nbr_blk, dp.sk_nbr_blk, P.sk_nbr_blk);
    upload(L.s_order, P.wave_order, s);
    L.s_rank.alloc(std::max(nsk, 1) * sizeof(int), s, true);
    L.s_rows.alloc(std::max(nsk, 1) * sizeof(int), s, true);
    upload(L.s_T_off, T_off, s);
    upload(L.s_P_off, SP_off, s);
    upload(L.s_work_off, work_off, s);
    upload(L.s_iwork_off, iwork_off, s);
    F->red.alloc(std::max<size_t>(G.mem.size(), 1), s, true);
    DBuf wk, iwk;
    wk.alloc(std::max<int64_t>(work, 1) * sizeof(double), s);
    iwk.alloc(std::max<int64_t>(iwork, 1) * sizeof(int), s);
    SkelArgs ka;
    ka.nsk = nsk;
    ka.groups = L.s_groups.as<int>();
    ka.nbr_off = L.s_nbr_off.as<int64_t>();
    ka.nbr = L.s_nbr.as<int>();
    ka.nbr_blk = L.s_nbr_blk.as<int>();
    ka.alive = F->alive.as<int>();
    ka.red = F->red.as<uint8_t>();
    ka.rank = L.s_rank.as<int>();
    ka.rows = L.s_rows.as<int>();
    ka.eps = F->eps;
    {
      // Gram-path ID when the ID tolerance leaves room for the squared conditioning of A^T A
      // (the rank cut sits far above sqrt(k eps_mach)); PHIF_GID=0 keeps Householder CPQR
      static const bool gid_on = !getenv("PHIF_GID") || atoi(getenv("PHIF_GID")) != 0;
      static const double gid_eps = getenv("PHIF_GID_EPS") ? atof(getenv("PHIF_GID_EPS")) : 1e-5;
      ka.gram = (gid_on && F->eps >= gid_eps) ? 1 : 0;
      ka.prof = gid_prof_buffer();
    }
    ka.work = wk.as<double>();
    ka.work_off = L.s_work_off.as<int64_t>();
    ka.iwork = iwk.as<int>();
    ka.iwork_off = L.s_iwork_off.as<int64_t>();
    ka.rec = L.rec.as<double>();
    ka.T_off = L.s_T_off.as<int64_t>();
    ka.P_off = L.s_P_off.as<int64_t>();
    if (timing) CK(cudaEventRecord(ev[8], s));
    for (int t = 0; t < nsk; ++t)
      if (P.sk_nbr_off[t + 1] - P.sk_nbr_off[t] > 256)
        throw std::runtime_error("skeletonize: a separator couples to more than 256 groups");
    // large separators: team / Gram-path ID; the rest one CTA each (thresholds env-tunable)
    static const int large_k = getenv("PHIF_LARGE_K") ? atoi(getenv("PHIF_LARGE_K")) : 48;
    static const int64_t large_mk = getenv("PHIF_LARGE_MK") ? atoll(getenv("PHIF_LARGE_MK")) : 100000;
    auto is_large = [&](int t) {
      const int kk = G.size(P.skeleton[t]);
      return kk > large_k && rows_bound[t] * kk > large_mk;
    };
    bool any_large = false;
    for (int t = 0; t < nsk; ++t)
      if (is_large(t)) any_large = true;
    static const bool no_dyn = getenv("PHIF_NO_DYN") != nullptr;
    if (nsk && !any_large && !no_dyn) {
      // only small separators: one persistent dependency-driven launch instead of per-wave launches
      DBuf nd, so, sc, done, next;
      dev_arr(nd, dp.sk_ndep, P.sk_ndep);
      dev_arr(so, dp.sk_succ_off, P.sk_succ_off);
      dev_arr(sc, dp.sk_succ, P.sk_succ);
      done.alloc(std::max(nsk, 1) * sizeof(int), s, true);
      next.alloc(sizeof(int), s, true);
      DynSched ds;
      ds.count = nsk;
      ds.next = next.as<int>();
      ds.done = done.as<int>();
      ds.ndep = nd.as<int>();
      ds.succ_off = so.as<int64_t>();
      ds.succ = sc.as<int>();
      ka.order = L.s_order.as<int>();
      int64_t need = 0;
      int sep_kmax = 0;
      for (int t = 0; t < nsk; ++t) {
        const int64_t kk = G.size(P.skeleton[t]);
        need = std::max<int64_t>(need, std::max<int64_t>(rows_bound[t], 1) * kk + 4 * kk + 4);
        sep_kmax = std::max(sep_kmax, (int)kk);
      }
      launch_skel_id_dyn(dv, ka, ds, need, s, sep_kmax);
      CK(cudaGetLastError());
      // (stream-ordered: no host sync needed here; buffers are recycled on the same stream)
    } else {
      // per wave: small separators -> one CTA each; large ones -> gather + team CPQR
      static int num_sms = 0;
      if (!num_sms) CK(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, 0));
      std::vector<int> small_list, large_list, team_face, team_off_all;
      std::vector<int64_t> small_off(P.nwaves + 1, 0), large_off(P.nwaves + 1, 0), toff_off(P.nwaves + 1, 0),
          slot_off(P.nwaves + 1, 0);
      std::vector<int> wave_blocks(P.nwaves, 0), wave_vcap(P.nwaves, 0), wave_kmax(P.nwaves, 0), wave_mmax(P.nwaves, 0);
      std::vector<int> wave_cluster(P.nwaves, 0);
      // Gram-path ID (gram_id.cuh) for the large separators under the same rule
      const bool use_gid = ka.gram != 0;
      std::vector<int> gid_item, gid_wi, gid_wj, gid_wit;
      std::vector<int64_t> gid_ld, gid_goff, gid_coff, gid_item_off(P.nwaves + 1, 0), gid_w_off(P.nwaves + 1, 0);
      std::vector<int> gid_C(P.nwaves, 1), gid_kmax(P.nwaves, 0), gid_P(P.nwaves, 1), gid_S(P.nwaves, 1);
      std::vector<uint8_t> gid_sg(P.nwaves, 0);
      int64_t gid_gbuf = 1, gid_cnt = 1, gid_go = 0, gid_co = 0;   // (R of every item persists until k_gid_T)
      int gid_kmax_lv = 0, gid_C_lv = 1;
      for (int w = 0; w < P.nwaves; ++w) {
        std::vector<int> large;
        for (int64_t q = P.wave_off[w]; q < P.wave_off[w + 1]; ++q) {
          const int t = P.wave_order[q];
          const int k = G.size(P.skeleton[t]);
          if (is_large(t)) {
            if (use_gid && gid_fits(k)) gid_item.push_back(t);
            else large.push_back(t);
          } else {
            small_list.push_back(t);
          }
        }
        gid_item_off[w + 1] = (int64_t)gid_item.size();
        gid_w_off[w] = (int64_t)gid_wi.size();
        {
          int kmx = 0;
          for (int64_t q = gid_item_off[w]; q < gid_item_off[w + 1]; ++q)
            kmx = std::max(kmx, G.size(P.skeleton[gid_item[q]]));
          gid_kmax[w] = kmx;
          const int ni = (int)(gid_item_off[w + 1] - gid_item_off[w]);
          if (ni) {
            bool sg = false;
            gid_C[w] = gid_cluster(kmx, &sg);
            gid_sg[w] = sg;
            gid_P[w] = std::max(1, std::min(32, 2 * num_sms / ni));
            gid_cnt = std::max<int64_t>(gid_cnt, (int64_t)ni * gid_P[w]);
          }
          // split-K of the Gram tiles so that a wave fills the GPU (partial blocks, fixed-order sum)
          int64_t ntiles = 0, rmin = INT64_MAX;
          for (int64_t q = gid_item_off[w]; q < gid_item_off[w + 1]; ++q) {
            const int t = gid_item[q], nt = (G.size(P.skeleton[t]) + 63) / 64;
            ntiles += (int64_t)nt * (nt + 1) / 2;
            rmin = std::min<int64_t>(rmin, rows_bound[t]);
          }
          static const int smax = env_int("PHIF_GID_SPLITK", 4);
          int S = 1;
          while (S < smax && ntiles * S < 2 * num_sms && rmin / (2 * S) >= 256) S *= 2;
          gid_S[w] = S;
          int64_t& go = gid_go;
          if (ni) {
            gid_kmax_lv = std::max(gid_kmax_lv, kmx);
            gid_C_lv = std::max(gid_C_lv, gid_C[w]);
          }
          for (int64_t q = gid_item_off[w]; q < gid_item_off[w + 1]; ++q) {
            const int t = gid_item[q];
            const int k = G.size(P.skeleton[t]);
            gid_ld.push_back(std::max<int64_t>(rows_bound[t], 1));
            gid_goff.push_back(go);
            gid_coff.push_back(gid_co);
            gid_co += k;
            go += gid_gbuf_doubles(k, gid_C[w], gid_sg[w], S);
            const int nt = (k + 63) / 64;
            for (int ks = 0; ks < S; ++ks)
              for (int it = 0; it < nt; ++it)
                for (int jt = 0; jt <= it; ++jt) {
                  gid_wit.push_back((int)(q - gid_item_off[w]));
                  gid_wi.push_back(it);
                  gid_wj.push_back(jt | (ks << 16));
                }
          }
          gid_gbuf = std::max(gid_gbuf, go);
        }
        gid_w_off[w + 1] = (int64_t)gid_wi.size();
        small_off[w + 1] = (int64_t)small_list.size();
        int vcap = 0, kmax = 0;
        double wsum = 0.0;
        for (int t : large) {
          kmax = std::max(kmax, G.size(P.skeleton[t]));
          wave_mmax[w] = std::max<int>(wave_mmax[w], (int)rows_bound[t]);
          vcap = std::max<int>(vcap, (int)std::min<int64_t>(rows_bound[t], 16384));
          wsum += (double)rows_bound[t] * G.size(P.skeleton[t]) * G.size(P.skeleton[t]);
        }
        int budget = large.empty() ? 0 : team_blocks_per_sm(vcap, kmax, team_colcap(vcap, kmax)) * num_sms;
        budget = std::max<int>(budget, (int)large.size());
        toff_off[w] = (int64_t)team_off_all.size();
        team_off_all.push_back(0);
        // team size: one owned-column chunk (16) per CTA when the budget allows, else work-proportional
        std::vector<int> want(large.size());
        int want_sum = 0;
        for (size_t q = 0; q < large.size(); ++q) {
          const int k = G.size(P.skeleton[large[q]]);
          want[q] = std::min(128, std::max(1, (k + 15) / 16));
          want_sum += want[q];
        }
        std::vector<int> Pv(large.size());
        int tot = 0;
        for (size_t q = 0; q < large.size(); ++q) {
          const int t = large[q];
          const int k = G.size(P.skeleton[t]);
          int Pf = want[q];
          if (want_sum > budget) {
            const double wf = (double)rows_bound[t] * k * k;
            Pf = std::max(1, std::min(want[q], (int)(budget * wf / wsum)));
          }
          Pv[q] = std::max(Pf, (k + 511) / 512);
          tot += Pv[q];
        }
        while (tot > budget) {   // trim the largest teams until the wave is co-resident
          size_t qm = std::max_element(Pv.begin(), Pv.end()) - Pv.begin();
          if (Pv[qm] <= (G.size(P.skeleton[large[qm]]) + 511) / 512) throw std::runtime_error("team CPQR: wave too large");
          --Pv[qm];
          --tot;
        }
        // thread-block clusters as teams when every face of the wave gets a co-resident cluster
        // of comparable size (cluster barriers instead of the global-memory team barrier)
        if (!large.empty()) {
          static const char* tmode = getenv("PHIF_TEAM_MODE");   // "coop" | "cluster" | auto
          const bool force_cl = tmode && !strcmp(tmode, "cluster"), no_cl = tmode && !strcmp(tmode, "coop");
          const double pmean = (double)tot / large.size();
          int csel = 0;
          if (!no_cl)
            for (int C : {16, 8, 4, 2}) {
              static std::map<std::pair<size_t, int>, int> cache;
              const auto key = std::make_pair((size_t)vcap * 100003 + kmax, C);
              auto itc = cache.find(key);
              if (itc == cache.end())
                itc = cache.emplace(key, team_max_clusters(vcap, kmax, team_colcap(vcap, kmax), C)).first;
              if (itc->second >= (int)large.size()) {
                if (force_cl || C >= pmean) csel = C;
                break;
              }
            }
          wave_cluster[w] = csel;
          if (csel) {
            for (auto& pv : Pv) pv = csel;
            tot = csel * (int)large.size();
          }
        }
        tot = 0;
        for (size_t q = 0; q < large.size(); ++q) {
          tot += Pv[q];
          team_face.push_back(large[q]);
          team_off_all.push_back(tot);
          large_list.push_back(large[q]);
        }
        large_off[w + 1] = (int64_t)large_list.size();
        L.team_P_mean += tot;
        slot_off[w + 1] = slot_off[w] + tot;
        wave_blocks[w] = tot;
        wave_vcap[w] = vcap;
        wave_kmax[w] = kmax;
      }
      L.n_large = (int)large_list.size();
      if (L.n_large) L.team_P_mean /= L.n_large;
      DBuf d_gitem, d_gld, d_goff, d_gcoff, d_gcol, d_gwit, d_gwi, d_gwj, d_gcnt, d_gbuf;
      if (!gid_item.empty()) {
        upload(d_gitem, gid_item, s);
        upload(d_gld, gid_ld, s);
        upload(d_goff, gid_goff, s);
        upload(d_gcoff, gid_coff, s);
        d_gcol.alloc(std::max<int64_t>(gid_co, 1) * sizeof(int), s);
        upload(d_gwit, gid_wit, s);
        upload(d_gwi, gid_wi, s);
        upload(d_gwj, gid_wj, s);
        d_gcnt.alloc(gid_cnt * sizeof(int), s);
        d_gbuf.alloc(gid_gbuf * sizeof(double), s);
      }
      L.n_gid = (int)gid_item.size();
      DBuf d_small, d_large, d_toff, hdr, sv, si;
      upload(d_small, small_list, s);
      upload(d_large, large_list, s);
      upload(d_toff, team_off_all, s);
      hdr.alloc(std::max<size_t>(large_list.size(), 1) * sizeof(TeamHdr), s, true);
      sv.alloc(std::max<int64_t>(2 * slot_off[P.nwaves], 1) * sizeof(double), s);
      int64_t cand_ld = 1;
      for (int w = 0; w < P.nwaves; ++w) cand_ld = std::max<int64_t>(cand_ld, wave_mmax[w]);
      int64_t max_blocks = 1;
      for (int w = 0; w < P.nwaves; ++w) max_blocks = std::max<int64_t>(max_blocks, wave_blocks[w]);
      DBuf cand;
      cand.alloc((size_t)2 * max_blocks * cand_ld * sizeof(double), s);
      int kmax_lv = 0;
      for (int w = 0; w < P.nwaves; ++w) kmax_lv = std::max(kmax_lv, wave_kmax[w]);
      const int64_t qt_ld = 8 * (int64_t)kmax_lv + 64;   // T factors of all QR panels of one face
      DBuf qtb;
      qtb.alloc(std::max<size_t>(large_list.size(), 1) * qt_ld * sizeof(double), s);
      si.alloc(std::max<int64_t>(2 * slot_off[P.nwaves], 1) * sizeof(int), s);
      for (int w = 0; w < P.nwaves; ++w) {
        ka.order = d_small.as<int>() + small_off[w];
        int64_t need = 0;
        for (int64_t q = small_off[w]; q < small_off[w + 1]; ++q) {
          const int t = small_list[q];
          const int64_t kk = G.size(P.skeleton[t]);
          need = std::max<int64_t>(need, std::max<int64_t>(rows_bound[t], 1) * kk + 4 * kk + 4);
        }
        launch_skel_id(dv, ka, (int)(small_off[w + 1] - small_off[w]), need, s);
        const int ng = (int)(gid_item_off[w + 1] - gid_item_off[w]);
        if (ng) {
          GramArgs ga;
          ga.nitem = ng;
          ga.item_sep = d_gitem.as<int>() + gid_item_off[w];
          ga.item_ld = d_gld.as<int64_t>() + gid_item_off[w];
          ga.P = gid_P[w];
          ga.cnt = d_gcnt.as<int>();
          ga.gbuf = d_gbuf.as<double>();
          ga.g_off = d_goff.as<int64_t>() + gid_item_off[w];
          ga.col = d_gcol.as<int>();
          ga.c_off = d_gcoff.as<int64_t>() + gid_item_off[w];
          ga.CT = 1;
          ga.tcap = 0;
          ga.w_item = d_gwit.as<int>() + gid_w_off[w];
          ga.w_i = d_gwi.as<int>() + gid_w_off[w];
          ga.w_j = d_gwj.as<int>() + gid_w_off[w];
          ga.nwork = (int)(gid_w_off[w + 1] - gid_w_off[w]);
          ga.C = gid_C[w];
          ga.S = gid_S[w];
          ga.prof = gid_prof_buffer();
          launch_gid(dv, ka, ga, gid_kmax[w], gid_sg[w] != 0, s);
        }
        const int nl = (int)(large_off[w + 1] - large_off[w]);
        if (nl) {
          TeamArgs ta;
          ta.nface = nl;
          ta.face = d_large.as<int>() + large_off[w];
          ta.team_off = d_toff.as<int>() + toff_off[w];
          ta.hdr = hdr.as<TeamHdr>() + large_off[w];
          ta.slot_v = sv.as<double>() + 2 * slot_off[w];
          ta.slot_i = si.as<int>() + 2 * slot_off[w];
          ta.vcap = wave_vcap[w];
          ta.kmax = wave_kmax[w];
          ta.cand = cand.as<double>();
          ta.cand_ld = cand_ld;
          ta.colcap = team_colcap(wave_vcap[w], wave_kmax[w]);
          ta.qt = qtb.as<double>() + large_off[w] * qt_ld;
          ta.qt_ld = qt_ld;
          ta.cluster = wave_cluster[w];
          ta.prof = team_prof_buffer();
          launch_skel_team(dv, ka, ta, wave_blocks[w], s);
        }
      }
      if (!gid_item.empty()) {
        // T = R11^-1 R12 of every Gram-path separator of the level, off the wave chain
        GramArgs ga{};
        ga.nitem = (int)gid_item.size();
        ga.item_sep = d_gitem.as<int>();
        ga.gbuf = d_gbuf.as<double>();
        ga.g_off = d_goff.as<int64_t>();
        ga.col = d_gcol.as<int>();
        ga.c_off = d_gcoff.as<int64_t>();
        ga.CT = gid_C_lv;
        ga.tcap = gid_T_cap(gid_kmax_lv);
        launch_gid_T(dv, ka, ga, gid_kmax_lv, s);
      }
      CK(cudaGetLastError());
      // (stream-ordered: no host sync needed here; buffers are recycled on the same stream)
    }
    // ranks and redundant flags back to the host (large separator updates, next level planning)
    L.h_rank.resize(nsk);
    std::vector<int> h_rows(nsk);
    std::vector<uint8_t> red(G.mem.size());
    if (nsk) CK(cudaMemcpyAsync(L.h_rank.data(), L.s_rank.p, nsk * sizeof(int), cudaMemcpyDeviceToHost, s));
    if (nsk) CK(cudaMemcpyAsync(h_rows.data(), L.s_rows.p, nsk * sizeof(int), cudaMemcpyDeviceToHost, s));
    if (!red.empty()) CK(cudaMemcpyAsync(red.data(), F->red.p, red.size(), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (timing) CK(cudaEventRecord(ev[9], s));
    DBG("level %d: skeleton update nsk=%d waves=%d", lev, nsk, P.nwaves);
    // survivors per member position, and the next level's plan completed with them on a host
    // thread while the skeleton updates are launched and run
    alive_mem.assign(G.mem.size(), 0);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int g = 0; g < G.G; ++g)
      if (G.kind[g] != 0)
        for (int64_t q = G.off[g]; q < G.off[g + 1]; ++q) alive_mem[q] = red[q] ? 0 : 1;
    if (preplan.valid())
      fin_task = std::async(std::launch::async, [&sp, &L, &alive_mem, pf = std::move(preplan)]() mutable {
        omp_set_num_threads(std::max(2, omp_get_num_procs() / 2));
        LevelPlan pp = pf.get();
        const bool ok = finish_preplan(sp, pp, L.plan, alive_mem);
        return std::make_pair(std::move(pp), ok);
      });
    {
      // zeroing + elimination of the redundant DOFs: one CTA per small separator, large ones
      // (kt >= BIG_N) through gather -> batched GEMMs -> tile Cholesky of the panel -> A_ss -= U
      std::vector<int> usmall, ubig;
      for (int t = 0; t < nsk; ++t) {
        const int kt = G.size(P.skeleton[t]) - L.h_rank[t];
        if (kt == 0) continue;
        (kt >= BIG_SEP ? ubig : usmall).push_back(t);
      }
      DBuf dus;
      upload(dus, usmall, s);
      launch_skel_update(dv, ka, dus.as<int>(), (int)usmall.size(), F->status.as<DevStatus>(), s);
      if (!ubig.empty()) {
        const int nb = (int)ubig.size();
        std::vector<int> idx, cn(nsk, 0), cb(nsk, 0);
        std::vector<int64_t> idx_off(nb), U_off_all(nsk, 0), U_off(nb);
        int64_t uacc = 0;
        std::vector<GemmDesc> d1, d2, d3;
        std::vector<int> w1d, w1t, w2d, w2t, w3d, w3t;
        double* rec0 = L.rec.as<double>();
        double* wk0 = ka.work;
        for (int q = 0; q < nb; ++q) {
          const int t = ubig[q], g = P.skeleton[t], k = G.size(g), r = L.h_rank[t], kt = k - r;
          idx_off[q] = (int64_t)idx.size();
          for (int j = 0; j < k; ++j)
            if (!red[G.off[g] + j]) idx.push_back(j);
          for (int j = 0; j < k; ++j)
            if (red[G.off[g] + j]) idx.push_back(j);
          cn[t] = kt;
          cb[t] = r;
          U_off_all[t] = U_off[q] = uacc;
          uacc += (int64_t)r * r;
          if (r > 0) {
            double* Ass = wk0 + work_off[t];
            double* Asr = Ass + (int64_t)r * r;
            double* Pn = rec0 + SP_off[t];
            double* Ast = Pn + (int64_t)kt * kt;
            const double* T = rec0 + T_off[t];
            auto add = [&](std::vector<GemmDesc>& d, std::vector<int>& wd, std::vector<int>& wt, GemmDesc gd) {
              for (int tt = 0; tt < (gd.M + 63) / 64; ++tt) {
                wd.push_back((int)d.size());
                wt.push_back(tt);
              }
              d.push_back(gd);
            };
            add(d1, w1d, w1t, GemmDesc{Ass, T, Ast, r, kt, r, r, kt, kt, 0, -1.0, 1.0});    // A~_st = A_sr - A_ss T
            add(d2, w2d, w2t, GemmDesc{T, Ast, Pn, kt, kt, r, kt, kt, kt, 1, -1.0, 1.0});   // A_tt -= T^T A~_st
            add(d3, w3d, w3t, GemmDesc{Asr, T, Pn, kt, kt, r, kt, kt, kt, 1, -1.0, 1.0});   // A_tt -= A_sr^T T
          }
        }
        DBuf dbig, didx, didx_off, dU, dU_off, g1, g2, g3, v1d, v1t, v2d, v2t, v3d, v3t;
        upload(dbig, ubig, s);
        upload(didx, idx, s);
        upload(didx_off, idx_off, s);
        upload(dU_off, U_off, s);
        dU.alloc(std::max<int64_t>(uacc, 1) * sizeof(double), s);
        launch_skel_big_gather(dv, ka, dbig.as<int>(), didx.as<int>(), didx_off.as<int64_t>(), nb, s);
        upload(g1, d1, s);
        upload(g2, d2, s);
        upload(g3, d3, s);
        upload(v1d, w1d, s);
        upload(v1t, w1t, s);
        upload(v2d, w2d, s);
        upload(v2t, w2t, s);
        upload(v3d, w3d, s);
        upload(v3t, w3t, s);
        launch_bgemm(g1.as<GemmDesc>(), v1d.as<int>(), v1t.as<int>(), (int)w1d.size(), s);
        launch_bgemm(g2.as<GemmDesc>(), v2d.as<int>(), v2t.as<int>(), (int)w2d.size(), s);
        launch_bgemm(g3.as<GemmDesc>(), v3d.as<int>(), v3t.as<int>(), (int)w3d.size(), s);
        BigPlan bps;
        bps.build(ubig, cn, cb, rec0, SP_off, dU.as<double>(), U_off_all, s);
        bps.run(F->status.as<DevStatus>(), s);
        launch_skel_big_post(dv, ka, dbig.as<int>(), didx.as<int>(), didx_off.as<int64_t>(), dU.as<double>(),
                             dU_off.as<int64_t>(), nb, s);
        CK(cudaStreamSynchronize(s));
      }
    }
    if (timing) CK(cudaEventRecord(ev[10], s));
    check_status(*F, lev, ST_SKELETONIZE);
    DBG("level %d: skeleton update done", lev);
    CK(cudaStreamSynchronize(s));
    if (getenv("PHIF_DUMP_SEP")) {
      FILE* fp = fopen(getenv("PHIF_DUMP_SEP"), lev == 0 ? "w" : "a");
      if (fp) {
        for (int t = 0; t < nsk; ++t)
          fprintf(fp, "%d %d %d %d %d\n", lev, P.sk_wave[t], G.size(P.skeleton[t]), h_rows[t], L.h_rank[t]);
        fclose(fp);
      }
    }
    tp = clk::now();
    // skeleton apply descriptors and the ID statistics: only the apply and the stats need them,
    // so they are built (and uploaded) on a host thread while the next level is planned and
    // factored; joined after the level loop (and before a level is dropped on NotSpd)
    {
      auto redp = std::make_shared<std::vector<uint8_t>>(std::move(red));
      auto rowsp = std::make_shared<std::vector<int>>(std::move(h_rows));
      auto pnp = std::make_shared<std::vector<int>>(std::move(pn));
      LevelRT* Lp = &L;
      int cur_dev = 0;
      CK(cudaGetDevice(&cur_dev));
      L.ap_task = std::async(std::launch::async, [Lp, redp, rowsp, pnp, nsk, r, s, cur_dev]() {
        CK(cudaSetDevice(cur_dev));   // (a new host thread starts on device 0)
        LevelRT& L = *Lp;
        const LevelPlan& P = L.plan;
        const Groups& G = P.grp;
        const std::vector<uint8_t>& red_t = *redp;
        const std::vector<int>& rows_t = *rowsp;
        const std::vector<int>& pn_t = *pnp;
        const std::vector<int64_t>& awork = L.h_awork;
        // skeleton apply descriptors (offsets by prefix sums, members filled in parallel)
        std::vector<int> sr(nsk), skt(nsk), Sd, Rd;
        std::vector<int64_t> S_off(nsk), R_off(nsk);
        int64_t rsum = 0, ktsum = 0;
        for (int t = 0; t < nsk; ++t) {
          const int g = P.skeleton[t];
          sr[t] = L.h_rank[t];
          skt[t] = G.size(g) - L.h_rank[t];
          S_off[t] = rsum;
          R_off[t] = ktsum;
          rsum += sr[t];
          ktsum += skt[t];
        }
        Sd.resize(rsum);
        Rd.resize(ktsum);
        for (int t = 0; t < nsk; ++t) {
          const int g = P.skeleton[t];
          int64_t a = S_off[t], b = R_off[t];
          for (int64_t q = G.off[g]; q < G.off[g + 1]; ++q) {
            if (red_t[q]) Rd[b++] = G.mem[q];
            else Sd[a++] = G.mem[q];
          }
        }
        for (int t = 0; t < nsk; ++t) {
          const double mm = rows_t[t], kk = sr[t] + skt[t], rr = sr[t], kt = skt[t];
          const double a = std::max(mm, kk), b = std::min(mm, kk);
          L.fl[3] += 2.0 * a * b * b - 2.0 * b * b * b / 3.0 + rr * rr * kt;   // GEQP3 + T solve
          L.by[3] += 8.0 * (mm * kk + rr * kt) + 4.0 * kk;
          if (kt > 0) {
            L.fl[4] += 2.0 * rr * rr * kt + 4.0 * rr * kt * kt + kt * kt * kt / 3.0 + kt * kt * rr + kt * rr * rr;
            L.by[4] += 8.0 * (kk * kk + rr * rr + (kt + rr) * kt + rr * kt);
          }
        }
        for (int t = 0; t < nsk; ++t) {
          const double kk = sr[t] + skt[t];
          L.sep_k_mean += kk / nsk;
          L.sep_m_mean += (double)rows_t[t] / nsk;
          L.sep_k_max = std::max(L.sep_k_max, kk);
          L.sep_m_max = std::max(L.sep_m_max, (double)rows_t[t]);
        }
        L.rho_max = nsk ? *std::max_element(sr.begin(), sr.end()) : 0;
        L.rho_mean = nsk ? (double)rsum / nsk : 0.0;
        upload(L.s_r, sr, s);
        upload(L.s_kt, skt, s);
        upload(L.s_S, Sd, s);
        upload(L.s_S_off, S_off, s);
        upload(L.s_R, Rd, s);
        upload(L.s_R_off, R_off, s);
        upload(L.s_awork_off, awork, s);
        L.h_S_off = S_off;
        L.h_R_off = R_off;
        L.h_sr = sr;
        L.h_skt = skt;
        {
          std::vector<int> small_sk, small_pr, tiny_sk;
          int tiny_rows = 1;
          for (int t = 0; t < nsk; ++t) {
            const int kk = G.size(P.skeleton[t]);
            if (skt[t] == 0 && kk < APPLY_BIG) continue;   // full rank: the record is the identity
            if (kk <= 64 && sr[t] > 0) {   // warp replay: rows r + 2 k~ staged per warp
              tiny_sk.push_back(t);
              tiny_rows = std::max(tiny_rows, sr[t] + 2 * skt[t]);
            } else if (kk < APPLY_BIG) {
              small_sk.push_back(t);
            }
          }
          L.n_apply_tiny_sk = (int)tiny_sk.size();
          L.apply_tiny_rows = tiny_rows;
          upload(L.d_apply_tiny_sk, tiny_sk, s);
          int pr_max = 1;
          for (int t = 0; t < r; ++t)
            if (pn_t[t] < APPLY_BIG) {
              small_pr.push_back(t);
              pr_max = std::max(pr_max, pn_t[t]);
            }
          L.apply_small_pr_max = pr_max;
          L.n_apply_small_sk = (int)small_sk.size();
          L.n_apply_small_pr = (int)small_pr.size();
          upload(L.d_apply_small_sk, small_sk, s);
          upload(L.d_apply_small_pr, small_pr, s);
        }
      });
    }
    plan_ms += ms_since(tp);
    L.t_ms[5] += ms_since(tp);
    DBG("level %d: next-level inputs ready", lev);
    L.t_wall_ms = ms_since(t_level0);
    if (timing) {
      CK(cudaEventSynchronize(ev[10]));
      float a;
      cudaEventElapsedTime(&a, ev[0], ev[1]); L.t_ms[0] = a;
      cudaEventElapsedTime(&a, ev[2], ev[3]); L.t_ms[1] = a;
      cudaEventElapsedTime(&a, ev[4], ev[5]); L.t_ms[1] += a;
      cudaEventElapsedTime(&a, ev[6], ev[7]); L.t_ms[2] = a;
      cudaEventElapsedTime(&a, ev[8], ev[9]); L.t_ms[3] = a;
      cudaEventElapsedTime(&a, ev[9], ev[10]); L.t_ms[4] = a;
    }
  }
  } catch (NotSpd& e) {
    // partial statistics: the levels completed before the failing one (errors.py:21-30)
    if (fin_task.valid()) fin_task.wait();   // (they read the plan of the level being dropped)
    if (preplan.valid()) preplan.wait();
    for (auto& lvp : F->levels)
      if (lvp->ap_task.valid()) lvp->ap_task.wait();
    cudaStreamSynchronize(s);
    while ((int)F->levels.size() > e.level) F->levels.pop_back();
    F->t_factor_ms = ms_since(t_start);
    F->t_plan_ms = plan_ms;
    e.partial = F->stats_json();
    if (timing)
      for (auto& ev1 : ev) cudaEventDestroy(ev1);
    throw;
  }
  for (auto& lvp : F->levels)
    if (lvp->ap_task.valid()) lvp->ap_task.get();
  CK(cudaStreamSynchronize(s));
  F->t_factor_ms = ms_since(t_start);
  for (auto& lvp : F->levels) {
    LevelRT& L = *lvp;
    if (!L.bd_task.valid()) continue;
    BdLists bl = L.bd_task.get();
    L.nbd = (int)bl.dof.size();
    upload(L.bd_dof, bl.dof, s);
    upload(L.bd_off, bl.off, s);
    upload(L.bd_rows, bl.rows, s);
  }
  CK(cudaStreamSynchronize(s));
  F->t_plan_ms = plan_ms;
  if (timing)
    for (auto& e : ev) cudaEventDestroy(e);
  F->red.release();
  return F;
}

// ---------------------------------------------------------------------------
// apply: mode 0 = F^-1 (up then down), 1 = G^-1 (up), 2 = G^-T (down)
// ---------------------------------------------------------------------------
static void ensure_work(Factorization& F, int k) {
  int64_t need = 1, needw = 1;
  for (auto& lp : F.levels) {
    need = std::max(need, std::max(lp->cell_work_unit, std::max(lp->prec_work_unit, lp->skel_work_unit)));
    needw = std::max(needw, lp->wbuf_unit);
  }
  const size_t wb = (size_t)need * k * sizeof(double), bb = (size_t)needw * k * sizeof(double);
  if (wb > F.work_cap) {
    F.work.alloc(wb, F.stream);
    F.work_cap = wb;
  }
  if (bb > F.wbuf_cap) {
    F.wbuf.alloc(bb, F.stream);
    F.wbuf_cap = bb;
  }
}

// gather/scatter segments are split so that one warp moves at most ~1024 values
static void push_seg(std::vector<int64_t>& src, std::vector<int64_t>& dst, std::vector<int>& len, int64_t s0,
                     int64_t d0, int n, int k) {
  const int step = std::max(1, 1024 / std::max(k, 1));
  for (int r = 0; r < n; r += step) {
    src.push_back(s0 + r);
    dst.push_back(d0 + r);
    len.push_back(std::min(step, n - r));
  }
}

// Order the work items [begin, end) of one replay-GEMM launch by decreasing K depth (stable): the
// persistent CTAs of k_rgemm take items w, w + G, w + 2G, ..., so every CTA gets one item of each
// depth tier (imbalance at most one item) and the shortest items fill the tail.
static void balance_items(std::vector<int>& wd, std::vector<int>& wt, size_t begin, size_t end,
                          const std::vector<GemmDesc>& d) {
  if (end - begin < 2) return;
  auto depth = [&](size_t i) {
    const GemmDesc& g = d[wd[i]];
    const int i0 = 64 * wt[i];
    if (g.tri == 1) return std::min(g.K, i0 + 64);
    if (g.tri == 3) return g.K - i0;
    return g.K;
  };
  std::vector<std::pair<int, size_t>> key(end - begin);
  for (size_t i = begin; i < end; ++i) key[i - begin] = {-depth(i), i};
  std::stable_sort(key.begin(), key.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
  std::vector<int> nd(end - begin), nt(end - begin);
  for (size_t j = 0; j < key.size(); ++j) {
    nd[j] = wd[key[j].second];
    nt[j] = wt[key[j].second];
  }
  std::copy(nd.begin(), nd.end(), wd.begin() + begin);
  std::copy(nt.begin(), nt.end(), wt.begin() + begin);
}

// GEMM replay of big cells: L^-T is stored below [L ; X^T] in the panel.
struct BigApply {
  int k = -1;
  double* work = nullptr;
  double* wbuf = nullptr;
  DBuf desc;                  // 4 phases of descriptors
  DBuf wd, wt;                // work lists (descriptor, row tile)
  int64_t ph_off[5] = {0, 0, 0, 0, 0};
  int ph_kmean[4] = {0, 0, 0, 0};   // mean K depth per work item of each phase
  DBuf gi_src, gi_dst, gi_len, sc_src, sc_dst, sc_len, gb_src, gb_dst, gb_len;
  int nbig = 0, nseg_i = 0, nseg_b = 0;
  void build(Factorization& F, LevelRT& L, int kk) {
    k = kk;
    work = F.work.as<double>();
    wbuf = F.wbuf.as<double>();
    cudaStream_t s = F.stream;
    const LevelPlan& P = L.plan;
    const double* rec = L.rec.as<double>();
    std::vector<GemmDesc> d;
    std::vector<int> wd_h, wt_h;
    std::vector<int64_t> isrc, idst, sdst, bsrc, bdst;
    std::vector<int> ilen, blen;
    int64_t ksum = 0;
    auto add = [&](const double* A, int lda, int ta, const double* B, double* C, int M, int K, double al,
                   double be, int tri) {
      if (M <= 0) return;
      ksum += (int64_t)((M + 63) / 64) * (tri ? (K + 1) / 2 : K);
      GemmDesc g;
      g.tri = tri;
      g.A = A;
      g.B = B;
      g.C = C;
      g.M = M;
      g.N = k;
      g.K = K;
      g.lda = lda;
      g.ldb = k;
      g.ldc = k;
      g.transA = ta;
      g.alpha = al;
      g.beta = be;
      const int id = (int)d.size();
      d.push_back(g);
      for (int t = 0; t < (M + 63) / 64; ++t) {
        wd_h.push_back(id);
        wt_h.push_back(t);
      }
    };
    std::vector<int> cells(P.interior.size());
    for (size_t t = 0; t < cells.size(); ++t) cells[t] = (int)t;
    nbig = (int)cells.size();
    // phase 0: Z = (L^-T)^T Y ; phase 1: W = X^T Z ; phase 2: Y -= X Xb ; phase 3: Z = L^-T Y
    for (int ph = 0; ph < 4; ++ph) {
      ph_off[ph] = (int64_t)wd_h.size();
      ksum = 0;
      for (int t : cells) {
        const int n = P.cell_n[t], b = P.cell_b[t];
        const double* Pp = rec + L.h_P_off[t];
        const double* XT = Pp + (int64_t)n * n;
        const double* LiT = Pp + (int64_t)(n + b) * n;
        double* Y = work + L.h_cwork[t] * k;
        double* Z = Y + (int64_t)n * k;
        double* Xb = Z + (int64_t)n * k;
        if (ph == 0) add(LiT, n, 1, Y, Z, n, n, 1.0, 0.0, 1);   // L^-1 = (L^-T)^T: lower
        if (ph == 1 && b > 0) add(XT, n, 0, Z, wbuf + L.h_B_off[t] * k, b, n, 1.0, 0.0, 0);
        if (ph == 2 && b > 0) add(XT, n, 1, Xb, Y, n, b, -1.0, 1.0, 0);
        if (ph == 3) add(LiT, n, 0, Y, Z, n, n, 1.0, 0.0, 3);   // L^-T: upper
      }
      ph_kmean[ph] = (int)(ksum / std::max<int64_t>(1, (int64_t)wd_h.size() - ph_off[ph]));
      balance_items(wd_h, wt_h, (size_t)ph_off[ph], wd_h.size(), d);
    }
    ph_off[4] = (int64_t)wd_h.size();
    std::vector<int64_t> ssrc;
    std::vector<int> slen;
    for (int t : cells) {
      const int n = P.cell_n[t], b = P.cell_b[t];
      push_seg(isrc, idst, ilen, L.h_I_off[t], L.h_cwork[t], n, k);
      push_seg(ssrc, sdst, slen, L.h_I_off[t], L.h_cwork[t] + n, n, k);
      if (b > 0) push_seg(bsrc, bdst, blen, L.h_B_off[t], L.h_cwork[t] + 2 * n, b, k);
    }
    nseg_i = (int)isrc.size();
    nseg_b = (int)bsrc.size();
    upload(sc_src, ssrc, s);
    upload(sc_len, slen, s);
    upload(desc, d, s);
    upload(wd, wd_h, s);
    upload(wt, wt_h, s);
    upload(gi_src, isrc, s);
    upload(gi_dst, idst, s);
    upload(gi_len, ilen, s);
    upload(sc_dst, sdst, s);
    upload(gb_src, bsrc, s);
    upload(gb_dst, bdst, s);
    upload(gb_len, blen, s);
  }
  void phase(int ph, cudaStream_t s) const {
    launch_rgemm(desc.as<GemmDesc>(), wd.as<int>() + ph_off[ph], wt.as<int>() + ph_off[ph],
                 (int)(ph_off[ph + 1] - ph_off[ph]), k, s, ph_kmean[ph]);
  }
  void up(LevelRT& L, double* x, cudaStream_t s) const {
    launch_rows(work, x, L.mem.as<int>(), gi_src.as<int64_t>(), gi_dst.as<int64_t>(), gi_len.as<int>(), nseg_i, k,
                false, s);
    phase(0, s);
    phase(1, s);
    launch_rows(work, x, L.mem.as<int>(), sc_src.as<int64_t>(), sc_dst.as<int64_t>(), sc_len.as<int>(), nseg_i, k,
                true, s);
  }
  void down(LevelRT& L, double* x, cudaStream_t s) const {
    launch_rows(work, x, L.mem.as<int>(), gi_src.as<int64_t>(), gi_dst.as<int64_t>(), gi_len.as<int>(), nseg_i, k,
                false, s);
    launch_rows(work, x, L.c_B.as<int>(), gb_src.as<int64_t>(), gb_dst.as<int64_t>(), gb_len.as<int>(), nseg_b, k,
                false, s);
    phase(2, s);
    phase(3, s);
    launch_rows(work, x, L.mem.as<int>(), sc_src.as<int64_t>(), sc_dst.as<int64_t>(), sc_len.as<int>(), nseg_i, k,
                true, s);
  }
};

static BigApply* big_apply(Factorization& F, LevelRT& L, int k) {
  if (L.plan.interior.empty()) return nullptr;
  if (!L.bigap) L.bigap = std::make_shared<BigApply>();
  BigApply& b = *L.bigap;
  if (b.k != k || b.work != F.work.as<double>() || b.wbuf != F.wbuf.as<double>()) b.build(F, L, k);
  return &b;
}

// GEMM replay of the big block-Jacobi and separator records of one level (explicit inverses
// stored below L and L~). Steps: gather rows -> batched GEMM phases -> scatter rows.
struct GemmReplay {
  int k = -1;
  double* work = nullptr;
  struct Step {
    int kind;      // 0 gather, 1 scatter, 2 gemm
    int64_t off, cnt;
    int idx;       // gather/scatter index array: 0 members, 1 skeleton DOFs, 2 redundant DOFs
                   // (GEMM steps: mean K depth per work item)
  };
  std::vector<Step> steps[4];   // 0 prec up, 1 prec down, 2 skel up, 3 skel down
  DBuf desc, wd, wt, ss, sd, sl;
  void build(Factorization& F, LevelRT& L, int kk) {
    k = kk;
    work = F.work.as<double>();
    const LevelPlan& P = L.plan;
    const Groups& G = P.grp;
    const double* rec = L.rec.as<double>();
    std::vector<GemmDesc> d;
    std::vector<int> wdh, wth;
    std::vector<int64_t> src, dst;
    std::vector<int> len;
    auto seg_begin = [&]() { return (int64_t)src.size(); };
    int64_t ksum = 0;
    auto add_step = [&](int which, int kind, int64_t off, int idx) {
      const int64_t cnt = (kind == 2 ? (int64_t)wdh.size() : (int64_t)src.size()) - off;
      if (cnt > 0) steps[which].push_back({kind, off, cnt, kind == 2 ? (int)(ksum / cnt) : idx});
      if (kind == 2) balance_items(wdh, wth, (size_t)off, wdh.size(), d);
      ksum = 0;
    };
    auto gemm = [&](const double* A, int lda, int ta, const double* B, double* C, int M, int K, double al,
                    double be) {
      if (M <= 0 || K <= 0) return;
      ksum += (int64_t)((M + 63) / 64) * K;
      GemmDesc g{A, B, C, M, k, K, lda, k, k, ta, al, be};
      const int id = (int)d.size();
      d.push_back(g);
      for (int t = 0; t < (M + 63) / 64; ++t) {
        wdh.push_back(id);
        wth.push_back(t);
      }
    };
    // ---- block Jacobi: x_g <- L^-1 x_g (up) / L^-T x_g (down)
    std::vector<int> bigp;
    if (F.method != 0 && !P.root)
      for (size_t t = 0; t < L.h_pn.size(); ++t)
        if (L.h_pn[t] >= APPLY_BIG) bigp.push_back((int)t);
    for (int dir = 0; dir < 2; ++dir) {
      int64_t o = seg_begin();
      for (int t : bigp) push_seg(src, dst, len, L.h_pI_off[t], L.h_pwork[t], L.h_pn[t], k);
      add_step(dir, 0, o, 0);
      o = (int64_t)wdh.size();
      for (int t : bigp) {
        const int n = L.h_pn[t];
        const double* LiT = rec + L.h_L_off[t] + (int64_t)n * n;
        double* Y = work + L.h_pwork[t] * k;
        gemm(LiT, n, dir == 0 ? 1 : 0, Y, Y + (int64_t)n * k, n, n, 1.0, 0.0);
      }
      add_step(dir, 2, o, 0);
      o = seg_begin();
      for (int t : bigp) push_seg(src, dst, len, L.h_pI_off[t], L.h_pwork[t] + L.h_pn[t], L.h_pn[t], k);
      add_step(dir, 1, o, 0);
    }
    // ---- separators: records [L~ ; X~^T ; L~^-T] and T
    std::vector<int> bigs;
    if (!P.root)
      for (size_t t = 0; t < P.skeleton.size(); ++t)
        if (G.size(P.skeleton[t]) >= APPLY_BIG && L.h_skt[t] > 0) bigs.push_back((int)t);
    for (int dir = 0; dir < 2; ++dir) {
      const int which = 2 + dir;
      int64_t o = seg_begin();
      for (int t : bigs) push_seg(src, dst, len, L.h_S_off[t], L.h_awork[t], L.h_sr[t], k);
      add_step(which, 0, o, 1);
      o = seg_begin();
      for (int t : bigs) push_seg(src, dst, len, L.h_R_off[t], L.h_awork[t] + L.h_sr[t], L.h_skt[t], k);
      add_step(which, 0, o, 2);
      for (int ph = 0; ph < 3; ++ph) {
        o = (int64_t)wdh.size();
        for (int t : bigs) {
          const int r = L.h_sr[t], kt = L.h_skt[t];
          const double* T = rec + L.h_T_off[t];
          const double* Pn = rec + L.h_SP_off[t];
          const double* PB = Pn + (int64_t)kt * kt;
          const double* LiT = Pn + (int64_t)(kt + r) * kt;
          double* Ys = work + L.h_awork[t] * k;
          double* Yr = Ys + (int64_t)r * k;
          double* Z = Yr + (int64_t)kt * k;
          if (dir == 0) {   // up: Yr -= T^T Ys ; Z = L~^-1 Yr ; Ys -= X~^T Z
            if (ph == 0) gemm(T, kt, 1, Ys, Yr, kt, r, -1.0, 1.0);
            if (ph == 1) gemm(LiT, kt, 1, Yr, Z, kt, kt, 1.0, 0.0);
            if (ph == 2) gemm(PB, kt, 0, Z, Ys, r, kt, -1.0, 1.0);
          } else {          // down: Yr -= X~ Ys ; Z = L~^-T Yr ; Ys -= T Z
            if (ph == 0) gemm(PB, kt, 1, Ys, Yr, kt, r, -1.0, 1.0);
            if (ph == 1) gemm(LiT, kt, 0, Yr, Z, kt, kt, 1.0, 0.0);
            if (ph == 2) gemm(T, kt, 0, Z, Ys, r, kt, -1.0, 1.0);
          }
        }
        add_step(which, 2, o, 0);
      }
      o = seg_begin();
      for (int t : bigs) push_seg(src, dst, len, L.h_S_off[t], L.h_awork[t], L.h_sr[t], k);
      add_step(which, 1, o, 1);
      o = seg_begin();
      for (int t : bigs) push_seg(src, dst, len, L.h_R_off[t], L.h_awork[t] + L.h_sr[t] + L.h_skt[t], L.h_skt[t], k);
      add_step(which, 1, o, 2);
    }
    cudaStream_t s = F.stream;
    upload(desc, d, s);
    upload(wd, wdh, s);
    upload(wt, wth, s);
    upload(ss, src, s);
    upload(sd, dst, s);
    upload(sl, len, s);
  }
  void run(int which, LevelRT& L, double* x, cudaStream_t s) const {
    for (const Step& st : steps[which]) {
      if (st.kind == 2) {
        launch_rgemm(desc.as<GemmDesc>(), wd.as<int>() + st.off, wt.as<int>() + st.off, (int)st.cnt, k, s, st.idx);
      } else {
        const int* idx = st.idx == 0 ? L.mem.as<int>() : (st.idx == 1 ? L.s_S.as<int>() : L.s_R.as<int>());
        launch_rows(work, x, idx, ss.as<int64_t>() + st.off, sd.as<int64_t>() + st.off, sl.as<int>() + st.off,
                    (int)st.cnt, k, st.kind == 1, s);
      }
    }
  }
};

static GemmReplay* gemm_replay(Factorization& F, LevelRT& L, int k) {
  if (!L.replay) L.replay = std::make_shared<GemmReplay>();
  GemmReplay& r = *L.replay;
  if (r.k != k || r.work != F.work.as<double>()) {
    r.steps[0].clear();
    r.steps[1].clear();
    r.steps[2].clear();
    r.steps[3].clear();
    r.build(F, L, k);
  }
  return &r;
}

static ApplyCellArgs cell_args(Factorization& F, LevelRT& L) {
  ApplyCellArgs a;
  a.list = nullptr;
  a.p = 0;   // every cell is replayed by batched GEMMs (big_apply)
  a.n = L.c_n.as<int>();
  a.b = L.c_b.as<int>();
  a.I = L.mem.as<int>();
  a.I_off = L.c_I_off.as<int64_t>();
  a.B = L.c_B.as<int>();
  a.B_off = L.c_B_off.as<int64_t>();
  a.rec = L.rec.as<double>();
  a.P_off = L.c_P_off.as<int64_t>();
  a.work = F.work.as<double>();
  a.work_off = L.c_work_off.as<int64_t>();
  a.wbuf = F.wbuf.as<double>();
  return a;
}

static ApplyPrecArgs prec_args(Factorization& F, LevelRT& L) {
  ApplyPrecArgs a;
  a.list = L.d_apply_small_pr.as<int>();
  a.r = (F.method != 0 && !L.plan.root) ? L.n_apply_small_pr : 0;
  a.ldn = L.apply_small_pr_max;
  a.n = L.p_n.as<int>();
  a.I = L.mem.as<int>();
  a.I_off = L.p_I_off.as<int64_t>();
  a.rec = L.rec.as<double>();
  a.L_off = L.p_L_off.as<int64_t>();
  a.work = F.work.as<double>();
  a.work_off = L.p_work_off.as<int64_t>();
  return a;
}

static ApplySkelArgs skel_args(Factorization& F, LevelRT& L) {
  ApplySkelArgs a;
  a.list = L.d_apply_small_sk.as<int>();
  a.nsk = L.plan.root ? 0 : L.n_apply_small_sk;
  a.r = L.s_r.as<int>();
  a.kt = L.s_kt.as<int>();
  a.S = L.s_S.as<int>();
  a.S_off = L.s_S_off.as<int64_t>();
  a.R = L.s_R.as<int>();
  a.R_off = L.s_R_off.as<int64_t>();
  a.rec = L.rec.as<double>();
  a.T_off = L.s_T_off.as<int64_t>();
  a.P_off = L.s_P_off.as<int64_t>();
  a.work = F.work.as<double>();
  a.work_off = L.s_awork_off.as<int64_t>();
  return a;
}

// forward replay G^T (up) / G (down) over every record (mode 3: F x = G G^T x, 4: G^T x, 5: G x)
static void apply_forward(Factorization& F, double* x, int k, int mode) {
  cudaStream_t s = F.stream;
  auto fwd_args = [&](LevelRT& L, ApplyCellArgs& c, ApplyPrecArgs& p, ApplySkelArgs& sk) {
    c = cell_args(F, L);
    c.p = (int)L.plan.interior.size();
    p = prec_args(F, L);
    p.list = nullptr;
    p.r = (F.method != 0 && !L.plan.root) ? (int)L.plan.precond.size() : 0;
    sk = skel_args(F, L);
    sk.list = nullptr;
    sk.nsk = L.plan.root ? 0 : (int)L.plan.skeleton.size();
  };
  if (mode == 3 || mode == 4) {
    for (auto& lp : F.levels) {
      LevelRT& L = *lp;
      ApplyCellArgs c;
      ApplyPrecArgs p;
      ApplySkelArgs sk;
      fwd_args(L, c, p, sk);
      launch_fwd(&c, nullptr, nullptr, x, k, true, s);
      if (L.plan.root) break;
      launch_fwd(nullptr, &p, nullptr, x, k, true, s);
      launch_fwd(nullptr, nullptr, &sk, x, k, true, s);
    }
  }
  if (mode == 3 || mode == 5) {
    for (int li = (int)F.levels.size() - 1; li >= 0; --li) {
      LevelRT& L = *F.levels[li];
      ApplyCellArgs c;
      ApplyPrecArgs p;
      ApplySkelArgs sk;
      fwd_args(L, c, p, sk);
      if (!L.plan.root) {
        launch_fwd(nullptr, nullptr, &sk, x, k, false, s);
        launch_fwd(nullptr, &p, nullptr, x, k, false, s);
      }
      launch_fwd(&c, nullptr, nullptr, x, k, false, s);
      launch_apply_reduce(L.bd_dof.as<int>(), L.bd_off.as<int64_t>(), L.bd_rows.as<int>(), F.wbuf.as<double>(),
                          L.nbd, x, k, s);
    }
  }
  CK(cudaGetLastError());
}

void apply(Factorization& F, double* x, int k, int mode) {
  ensure_work(F, k);
  cudaStream_t s = F.stream;
  if (mode >= 3) {
    apply_forward(F, x, k, mode);
    return;
  }
  if (mode == 0 || mode == 1) {
    for (auto& lp : F.levels) {
      LevelRT& L = *lp;
      launch_apply_cell(cell_args(F, L), x, k, true, s);
      if (apply_cell_mma_fits(L.cell_nmax, L.cell_bmax, k) && !L.plan.interior.empty()) {
        ApplyCellArgs c = cell_args(F, L);
        c.p = (int)L.plan.interior.size();
        launch_apply_cell_mma(c, L.cell_nmax, L.cell_bmax, x, true, s);
      } else if (BigApply* ba = big_apply(F, L, k)) {
        ba->up(L, x, s);
      }
      launch_apply_reduce(L.bd_dof.as<int>(), L.bd_off.as<int64_t>(), L.bd_rows.as<int>(), F.wbuf.as<double>(),
                          L.nbd, x, k, s);
      if (L.plan.root) break;
      GemmReplay* gr = gemm_replay(F, L, k);
      launch_apply_prec(prec_args(F, L), x, k, true, s);
      gr->run(0, L, x, s);
      launch_apply_skel(skel_args(F, L), x, k, true, s);
      launch_apply_skel_warp(skel_args(F, L), L.d_apply_tiny_sk.as<int>(), L.plan.root ? 0 : L.n_apply_tiny_sk, x, k, true,
                             L.apply_tiny_rows, s);
      gr->run(2, L, x, s);
    }
  }
  if (mode == 0 || mode == 2) {
    for (int li = (int)F.levels.size() - 1; li >= 0; --li) {
      LevelRT& L = *F.levels[li];
      if (!L.plan.root) {
        GemmReplay* gr = gemm_replay(F, L, k);
        launch_apply_skel(skel_args(F, L), x, k, false, s);
        launch_apply_skel_warp(skel_args(F, L), L.d_apply_tiny_sk.as<int>(), L.n_apply_tiny_sk, x, k, false,
                               L.apply_tiny_rows, s);
        gr->run(3, L, x, s);
        launch_apply_prec(prec_args(F, L), x, k, false, s);
        gr->run(1, L, x, s);
      }
      launch_apply_cell(cell_args(F, L), x, k, false, s);
      if (apply_cell_mma_fits(L.cell_nmax, L.cell_bmax, k) && !L.plan.interior.empty()) {
        ApplyCellArgs c = cell_args(F, L);
        c.p = (int)L.plan.interior.size();
        launch_apply_cell_mma(c, L.cell_nmax, L.cell_bmax, x, false, s);
      } else if (BigApply* ba = big_apply(F, L, k)) {
        ba->down(L, x, s);
      }
    }
  }
  CK(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// PCG: per-column scalars, converged columns frozen,
// true residual every 50 iterations, BreakdownError on non-finite values.
// ---------------------------------------------------------------------------
PcgResult pcg(const Matrix& A, Factorization* F, const double* b, double* x, int k, double tol, int maxit,
              cudaStream_t s, bool want_history) {
  // The per-column scalars, convergence flags and the residual history stay on the device; the
  // host reads two integers per iteration (active columns, breakdown) to stop the loop.
  const int64_t N = A.N;
  const size_t vb = (size_t)N * k * sizeof(double);
  DBuf R, Z, Pv, Q, part, sc, ctlb, hist;
  R.alloc(vb, s);
  Z.alloc(vb, s);
  Pv.alloc(vb, s);
  Q.alloc(vb, s);
  part.alloc((size_t)dot_part_blocks() * k * sizeof(double), s);
  sc.alloc(10 * (size_t)k * sizeof(double), s);
  double* rz = sc.as<double>();
  double* pq = rz + k;
  double* alpha = pq + k;
  double* beta = alpha + k;
  double* rn2 = beta + k;
  double* rzn = rn2 + k;
  double* bn2 = rzn + k;
  double* bn = bn2 + k;
  double* relres = bn + k;
  ctlb.alloc((3 * (size_t)k + 2) * sizeof(int), s);
  int* ctl = ctlb.as<int>();
  int* act = ctl + 2;
  int* iters = act + k;
  int* conv = iters + k;
  if (want_history && maxit > 0) hist.alloc((size_t)maxit * k * sizeof(double), s);
  double* hp = want_history && maxit > 0 ? hist.as<double>() : nullptr;
  PcgResult res;
  int hctl[2] = {0, 0};
  auto read_ctl = [&]() {
    CK(cudaMemcpyAsync(hctl, ctl, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  };
  CK(cudaMemsetAsync(x, 0, vb, s));
  CK(cudaMemcpyAsync(R.p, b, vb, cudaMemcpyDeviceToDevice, s));
  launch_dot(b, b, N, k, part.as<double>(), bn2, s);
  launch_pcg_init(bn2, bn, act, relres, iters, conv, ctl, k, s);
  auto precond = [&](double* dst, const double* src) {
    CK(cudaMemcpyAsync(dst, src, vb, cudaMemcpyDeviceToDevice, s));
    if (F) apply(*F, dst, k, 0);
  };
  precond(Z.as<double>(), R.as<double>());
  CK(cudaMemcpyAsync(Pv.p, Z.p, vb, cudaMemcpyDeviceToDevice, s));
  launch_dot(R.as<double>(), Z.as<double>(), N, k, part.as<double>(), rz, s);
  read_ctl();
  int it = 0;
  while (hctl[0] > 0 && it < maxit) {
    ++it;
    spmv(A, Pv.as<double>(), Q.as<double>(), k, s);
    launch_dot(Pv.as<double>(), Q.as<double>(), N, k, part.as<double>(), pq, s);
    launch_pcg_alpha(rz, pq, act, alpha, ctl, it, k, s);
    if (it % 50 == 0) {   // true residual
      launch_axpy(x, Pv.as<double>(), alpha, 1.0, act, N, k, s);
      spmv(A, x, Q.as<double>(), k, s);
      launch_sub(R.as<double>(), b, Q.as<double>(), act, N, k, s);
      launch_dot(R.as<double>(), R.as<double>(), N, k, part.as<double>(), rn2, s);
    } else {   // x += alpha p ; r -= alpha q ; ||r||^2 in one pass
      launch_pcg_update(x, Pv.as<double>(), R.as<double>(), Q.as<double>(), alpha, act, N, k, part.as<double>(), rn2,
                        s);
    }
    launch_pcg_check(rn2, bn, act, relres, iters, conv, hp, it, tol, ctl, k, s);
    read_ctl();
    if (hctl[1]) break;
    if (hctl[0] == 0) break;
    precond(Z.as<double>(), R.as<double>());
    launch_dot(R.as<double>(), Z.as<double>(), N, k, part.as<double>(), rzn, s);
    launch_pcg_beta(rzn, rz, act, beta, ctl, it, k, s);
    launch_xpby(Pv.as<double>(), Z.as<double>(), beta, act, N, k, s);
  }
  if (!hctl[1] && it > 0) read_ctl();   // (a breakdown flagged by the last beta)
  res.breakdown = hctl[1];
  res.iters.resize(k);
  res.relres.resize(k);
  res.converged.resize(k);
  CK(cudaMemcpyAsync(res.iters.data(), iters, k * sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(res.relres.data(), relres, k * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(res.converged.data(), conv, k * sizeof(int), cudaMemcpyDeviceToHost, s));
  res.history_len = hp ? it : 0;
  if (hp && it > 0) {
    res.history.resize((size_t)it * k);
    CK(cudaMemcpyAsync(res.history.data(), hp, (size_t)it * k * sizeof(double), cudaMemcpyDeviceToHost, s));
  }
  CK(cudaStreamSynchronize(s));
  return res;
}

// ---------------------------------------------------------------------------
// e_s = ||I - G^-1 A G^-T||_2 by power iteration
// ---------------------------------------------------------------------------
// power iteration ||op||_2 of a symmetric op from the host start vector x0 (oracle/diagnostics.py
// power_norm): x unit, y = op(x), estimate = |x^T y| (Rayleigh quotient),
// x <- y / ||y||; converged when successive Rayleigh quotients agree to rel_tol
template <typename Op>
static PowerResult power_norm_dev(int64_t N, cudaStream_t s, const double* x0, double rel_tol, int maxit, Op op) {
  DBuf X, Y, part, sc;
  X.alloc(N * sizeof(double), s);
  Y.alloc(N * sizeof(double), s);
  part.alloc(dot_part_blocks() * sizeof(double), s);
  sc.alloc(4 * sizeof(double), s);
  double* nrm2 = sc.as<double>();
  double* rq = nrm2 + 1;
  CK(cudaMemcpyAsync(X.p, x0, N * sizeof(double), cudaMemcpyHostToDevice, s));
  launch_dot(X.as<double>(), X.as<double>(), N, 1, part.as<double>(), nrm2, s);
  launch_scale(X.as<double>(), X.as<double>(), nrm2, N, s);
  PowerResult pr;
  double prev = -1.0;
  for (int it = 1; it <= maxit; ++it) {
    op(X.as<double>(), Y.as<double>());
    launch_dot(X.as<double>(), Y.as<double>(), N, 1, part.as<double>(), rq, s);   // Rayleigh quotient x^T op x
    launch_dot(Y.as<double>(), Y.as<double>(), N, 1, part.as<double>(), nrm2, s);
    double h[2];
    CK(cudaMemcpyAsync(h, nrm2, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const double est = std::fabs(h[1]);
    pr.iters = it;
    pr.value = est;
    if (h[0] == 0.0) {
      pr.value = 0.0;
      pr.converged = 1;
      pr.rel = 0.0;
      return pr;
    }
    if (prev >= 0.0) {
      pr.rel = est > 0.0 ? std::fabs(est - prev) / est : std::fabs(est - prev);
      if (pr.rel <= rel_tol) {
        pr.converged = 1;
        return pr;
      }
    }
    prev = est;
    launch_scale(X.as<double>(), Y.as<double>(), nrm2, N, s);
  }
  return pr;
}

// e_a = ||A - F|| / ||A||: two power iterations from the same start vector
PowerResult apply_error(const Matrix& A, Factorization& F, const double* x0, double rel_tol, int maxit) {
  cudaStream_t s = F.stream;
  const int64_t N = A.N;
  DBuf T;
  T.alloc(N * sizeof(double), s);
  PowerResult num = power_norm_dev(N, s, x0, rel_tol, maxit, [&](double* X, double* Y) {
    spmv(A, X, T.as<double>(), 1, s);   // T = A x
    CK(cudaMemcpyAsync(Y, X, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
    apply(F, Y, 1, 3);                   // Y = F x
    launch_xmy(Y, T.as<double>(), N, s);   // Y = A x - F x
  });
  PowerResult den = power_norm_dev(N, s, x0, rel_tol, maxit, [&](double* X, double* Y) {
    spmv(A, X, Y, 1, s);
  });
  PowerResult r;
  r.value = den.value > 0.0 ? num.value / den.value : 0.0;
  r.iters = num.iters + den.iters;
  r.converged = num.converged && den.converged;
  r.rel = std::max(num.rel, den.rel);
  return r;
}

// root block Cholesky factor B_L (n x n, row-major lower); returns n
int root_factor(Factorization& F, double* out) {
  LevelRT& R = *F.levels.back();
  if (R.plan.interior.empty()) return 0;
  const int n = R.plan.cell_n[0];
  if (out)
    CK(cudaMemcpyAsync(out, R.rec.as<double>() + R.h_P_off[0], (size_t)n * n * sizeof(double), cudaMemcpyDefault,
                       F.stream));
  CK(cudaStreamSynchronize(F.stream));
  return n;
}

PowerResult solve_error(const Matrix& A, Factorization& F, const double* x0, double rel_tol, int maxit) {
  cudaStream_t s = F.stream;
  const int64_t N = A.N;
  DBuf T;
  T.alloc(N * sizeof(double), s);
  return power_norm_dev(N, s, x0, rel_tol, maxit, [&](double* X, double* Y) {
    CK(cudaMemcpyAsync(T.p, X, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
    apply(F, T.as<double>(), 1, 2);   // G^-T x
    spmv(A, T.as<double>(), Y, 1, s);
    apply(F, Y, 1, 1);                // G^-1 A G^-T x
    launch_xmy(Y, X, N, s);           // x - G^-1 A G^-T x
  });
}

std::string Factorization::stats_json() const {
  std::ostringstream o;
  o.precision(17);
  const char* mname[] = {"hif", "phif", "exact"};
  o << "{\"method\":\"" << mname[method] << "\",\"eps\":" << eps << ",\"N\":" << spec.N << ",\"L\":" << spec.L
    << ",\"t_factor_ms\":" << t_factor_ms << ",\"t_plan_ms\":" << t_plan_ms << ",\"mem_bytes\":" << rec_bytes
    << ",\"levels\":[";
  for (size_t i = 0; i < levels.size(); ++i) {
    const LevelRT& L = *levels[i];
    const LevelPlan& P = L.plan;
    o << (i ? "," : "") << "{\"level\":" << P.level << ",\"S\":" << L.S << ",\"p\":" << P.interior.size()
      << ",\"q\":" << (P.root ? 0 : P.skeleton.size()) << ",\"r\":" << (P.root ? 0 : P.precond.size())
      << ",\"blocks\":" << P.pat.bg.size() << ",\"waves\":" << P.nwaves << ",\"rho_max\":" << L.rho_max
      << ",\"rho_mean\":" << L.rho_mean << ",\"sep_k_mean\":" << L.sep_k_mean << ",\"sep_k_max\":" << L.sep_k_max
      << ",\"sep_m_mean\":" << L.sep_m_mean << ",\"sep_m_max\":" << L.sep_m_max << ",\"n_large\":" << L.n_large << ",\"n_gid\":" << L.n_gid
      << ",\"cell_n_max\":" << (P.cell_n.empty() ? 0 : *std::max_element(P.cell_n.begin(), P.cell_n.end()))
      << ",\"cell_b_max\":" << (P.cell_b.empty() ? 0 : *std::max_element(P.cell_b.begin(), P.cell_b.end()))
      << ",\"team_P_mean\":" << L.team_P_mean << ",\"t_repack_ms\":" << L.t_ms[0] << ",\"t_eliminate_ms\":" << L.t_ms[1]
      << ",\"t_precondition_ms\":" << L.t_ms[2] << ",\"t_id_ms\":" << L.t_ms[3] << ",\"t_skel_update_ms\":"
      << L.t_ms[4] << ",\"t_plan_ms\":" << L.t_ms[5] << ",\"t_wall_ms\":" << L.t_wall_ms << ",\"t_host_overlap_ms\":" << L.t_host_overlap_ms << ",\"record_bytes\":" << L.rec_doubles * 8 << ",\"flops\":[" << L.fl[0] << "," << L.fl[1]
      << "," << L.fl[2] << "," << L.fl[3] << "," << L.fl[4] << "],\"bytes\":[" << L.by[0] << "," << L.by[1] << ","
      << L.by[2] << "," << L.by[3] << "," << L.by[4] << "]}";
  }
  const bool done = !levels.empty() && levels.back()->plan.root;
  o << "],\"SL\":" << (done && !levels.back()->plan.interior.empty() ? levels.back()->plan.cell_n[0] : 0)
    << ",\"complete\":" << (done ? "true" : "false") << "}";
  return o.str();
}

}  // namespace phif
