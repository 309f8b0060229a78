// extern "C" boundary (include/phif_b200.h). No exception crosses it.
#include <chrono>
#include <csignal>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <execinfo.h>
#include <unistd.h>

#include "../../include/phif_b200.h"
#include "engine.h"
#include "gpu_plan.h"
#include "problem.h"

struct phif_matrix {
  std::unique_ptr<phif::Matrix> m;
  cudaStream_t stream;
};
struct phif_factor {
  std::unique_ptr<phif::Factorization> f;
  // A finished factor is read-only, but its apply workspaces and lazily built replay plans are
  // per factor: concurrent callers are serialised here, each call synchronous.
  std::mutex mu;
};

namespace {

void segv_handler(int sig) {
  void* frames[64];
  const int n = backtrace(frames, 64);
  const char msg[] = "[phif] fatal signal, native backtrace:\n";
  if (write(2, msg, sizeof(msg) - 1) < 0) {}
  backtrace_symbols_fd(frames, n, 2);
  signal(sig, SIG_DFL);
  raise(sig);
}

struct InstallHandler {
  InstallHandler() {
    if (getenv("PHIF_DEBUG")) signal(SIGSEGV, segv_handler);
  }
} install_handler;

void set_err(phif_error* e, int code, const char* msg) {
  if (!e) return;
  e->code = code;
  e->pivot = e->level = e->stage = e->group = -1;
  std::snprintf(e->message, sizeof(e->message), "%s", msg);
}

thread_local std::string g_partial_stats;   // stats of the levels done before the last NotSpd

template <class Fn>
int guarded(phif_error* err, Fn&& fn) {
  try {
    fn();
    if (err) err->code = PHIF_OK;
    return PHIF_OK;
  } catch (const phif::NotSpd& e) {
    g_partial_stats = e.partial;
    if (err) {
      err->code = PHIF_NOT_SPD;
      err->pivot = e.pivot;
      err->level = e.level;
      err->stage = e.stage;
      err->group = e.group;
      std::snprintf(err->message, sizeof(err->message), "matrix not positive definite at pivot %d", e.pivot);
    }
    return PHIF_NOT_SPD;
  } catch (const std::exception& e) {
    set_err(err, PHIF_ERROR, e.what());
    return PHIF_ERROR;
  } catch (...) {
    set_err(err, PHIF_ERROR, "unknown error");
    return PHIF_ERROR;
  }
}

bool is_device(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace

extern "C" {

int phif_version(void) { return 1; }

long long phif_launch_count(void) { return phif::launch_count(); }

int phif_matrix_create(const int64_t* rowptr, const int32_t* col, const double* val, int64_t n, void* stream,
                       phif_matrix** out, phif_error* err) {
  return guarded(err, [&] {
    auto* A = new phif_matrix;
    A->stream = (cudaStream_t)stream;
    A->m = phif::matrix_create(rowptr, col, val, n, A->stream);
    cudaStreamSynchronize(A->stream);
    *out = A;
  });
}

void phif_matrix_free(phif_matrix* A) { delete A; }

int phif_matrix_from_field(int dim, int n, const double* a, const double* weights, int nweights, double lo, double hi,
                           double bh2, void* stream, phif_matrix** out, phif_error* err) {
  return guarded(err, [&] {
    if (dim < 2 || dim > 3 || n < 2) throw std::invalid_argument("phif_matrix_from_field: bad grid");
    cudaStream_t s = (cudaStream_t)stream;
    int64_t N = 1;
    for (int d = 0; d < dim; ++d) N *= (n - 1);
    phif::DBuf f;
    f.alloc(N * sizeof(double), s);
    if (is_device(a)) cudaMemcpyAsync(f.p, a, N * sizeof(double), cudaMemcpyDeviceToDevice, s);
    else phif::upload_bytes(f.p, a, N * sizeof(double), s);
    if (nweights > 0) {
      if (nweights % 2 != 1) throw std::invalid_argument("phif_matrix_from_field: odd number of weights expected");
      phif::smooth_field(dim, n - 1, f.as<double>(), std::vector<double>(weights, weights + nweights), s);
    }
    if (lo != 0.0 || hi != 0.0) phif::threshold_field(f.as<double>(), N, lo, hi, s);
    auto* A = new phif_matrix;
    A->stream = s;
    try {
      A->m = phif::matrix_from_field(dim, n, f.as<double>(), bh2, s, false);
    } catch (...) {
      delete A;
      throw;
    }
    *out = A;
  });
}

int phif_matrix_csr(const phif_matrix* A, int64_t* nnz, int64_t* rowptr, int32_t* col, double* val, double* field) {
  const phif::Matrix& M = *A->m;
  *nnz = M.nnz;
  if (rowptr) cudaMemcpy(rowptr, M.rowptr.p, (M.N + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost);
  if (col) cudaMemcpy(col, M.col.p, M.nnz * sizeof(int), cudaMemcpyDeviceToHost);
  if (val) cudaMemcpy(val, M.val.p, M.nnz * sizeof(double), cudaMemcpyDeviceToHost);
  if (field && M.stencil) cudaMemcpy(field, M.field.p, M.N * sizeof(double), cudaMemcpyDeviceToHost);
  return cudaGetLastError() == cudaSuccess ? PHIF_OK : PHIF_ERROR;
}

int phif_matrix_apply(const phif_matrix* A, const double* x, double* y, int nrhs, int force_csr, phif_error* err) {
  return guarded(err, [&] {
    const phif::Matrix& M = *A->m;
    cudaStream_t s = A->stream;
    const size_t bytes = (size_t)M.N * nrhs * sizeof(double);
    phif::DBuf dx, dy;
    dx.alloc(bytes, s);
    dy.alloc(bytes, s);
    phif::upload_bytes(dx.p, x, bytes, s);
    if (force_csr)
      phif::launch_spmv(M.rowptr.as<int64_t>(), M.col.as<int>(), M.val.as<double>(), dx.as<double>(), dy.as<double>(),
                        M.N, nrhs, s);
    else
      phif::spmv(M, dx.as<double>(), dy.as<double>(), nrhs, s);
    phif::download_bytes(y, dy.p, bytes, s);
    cudaStreamSynchronize(s);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw phif::CudaError(cudaGetErrorString(e));
  });
}

int phif_factorize(const phif_matrix* A, int dim, int n, int m, double eps, int method, void* stream, int timing,
                   phif_factor** out, phif_error* err) {
  return guarded(err, [&] {
    auto* F = new phif_factor;
    try {
      F->f = phif::factorize(*A->m, dim, n, m, eps, method, (cudaStream_t)stream, timing != 0);
    } catch (...) {
      delete F;
      throw;
    }
    *out = F;
  });
}

void phif_factor_free(phif_factor* F) { delete F; }

int phif_apply(phif_factor* F, double* x, int nrhs, int mode, phif_error* err) {
  return guarded(err, [&] {
    std::lock_guard<std::mutex> lock(F->mu);
    if (mode < 0 || mode > 5) throw std::invalid_argument("phif_apply: mode must be 0..5");
    phif::Factorization& f = *F->f;
    const size_t bytes = (size_t)f.spec.N * nrhs * sizeof(double);
    if (is_device(x)) {
      phif::apply(f, x, nrhs, mode);
      cudaStreamSynchronize(f.stream);
    } else {
      phif::DBuf d;
      d.alloc(bytes, f.stream);
      phif::upload_bytes(d.p, x, bytes, f.stream);
      phif::apply(f, d.as<double>(), nrhs, mode);
      phif::download_bytes(x, d.p, bytes, f.stream);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw phif::CudaError(cudaGetErrorString(e));
  });
}

int phif_pcg(const phif_matrix* A, phif_factor* F, const double* b, double* x, int nrhs, double tol, int maxit,
             void* stream, int* iters, double* relres, int* converged, double* history, int* history_len,
             phif_error* err) {
  int brk = 0;
  int rc = guarded(err, [&] {
    std::unique_lock<std::mutex> lock;
    if (F) lock = std::unique_lock<std::mutex>(F->mu);
    cudaStream_t s = F ? F->f->stream : (cudaStream_t)stream;
    const size_t bytes = (size_t)A->m->N * nrhs * sizeof(double);
    phif::DBuf db, dx;
    const double* bd = b;
    double* xd = x;
    const bool xdev = is_device(x);
    if (!is_device(b)) {
      db.alloc(bytes, s);
      phif::upload_bytes(db.p, b, bytes, s);
      bd = db.as<double>();
    }
    if (!xdev) {
      dx.alloc(bytes, s);
      xd = dx.as<double>();
    }
    phif::PcgResult r = phif::pcg(*A->m, F ? F->f.get() : nullptr, bd, xd, nrhs, tol, maxit, s, history != nullptr);
    if (history_len) *history_len = r.history_len;
    if (history && r.history_len) std::memcpy(history, r.history.data(), r.history.size() * sizeof(double));
    if (!xdev) phif::download_bytes(x, xd, bytes, s);
    cudaStreamSynchronize(s);
    for (int c = 0; c < nrhs; ++c) {
      if (iters) iters[c] = r.iters[c];
      if (relres) relres[c] = r.relres[c];
      if (converged) converged[c] = r.converged[c];
    }
    brk = r.breakdown;
  });
  if (rc == PHIF_OK && brk) {
    set_err(err, PHIF_BREAKDOWN, "non-finite PCG recurrence value");
    if (err) err->group = brk;
    return PHIF_BREAKDOWN;
  }
  return rc;
}

int phif_solve_error(const phif_matrix* A, phif_factor* F, const double* x0, double rel_tol, int maxit,
                     double* value, int* iters, int* converged, double* rel_achieved, phif_error* err) {
  return guarded(err, [&] {
    std::lock_guard<std::mutex> lock(F->mu);
    phif::PowerResult r = phif::solve_error(*A->m, *F->f, x0, rel_tol, maxit);
    *value = r.value;
    *iters = r.iters;
    *converged = r.converged;
    *rel_achieved = r.rel;
  });
}

int phif_apply_error(const phif_matrix* A, phif_factor* F, const double* x0, double rel_tol, int maxit,
                     double* value, int* iters, int* converged, double* rel_achieved, phif_error* err) {
  return guarded(err, [&] {
    std::lock_guard<std::mutex> lock(F->mu);
    phif::PowerResult r = phif::apply_error(*A->m, *F->f, x0, rel_tol, maxit);
    *value = r.value;
    *iters = r.iters;
    *converged = r.converged;
    *rel_achieved = r.rel;
  });
}

int phif_root_factor(phif_factor* F, double* out, int* n, phif_error* err) {
  return guarded(err, [&] {
    std::lock_guard<std::mutex> lock(F->mu);
    *n = phif::root_factor(*F->f, out);
  });
}

size_t phif_stats_json(const phif_factor* F, char* buf, size_t cap) {
  const std::string s = F->f->stats_json();
  if (buf && cap) {
    const size_t n = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return s.size();
}

int phif_plan_check(const phif_matrix* A, int dim, int n, int m, char* report, size_t cap) {
  std::string rep;
  int bad = 0;
  try {
    phif::Spec s;
    s.init(dim, n, m);
    const phif::Matrix& M = *A->m;
    M.ensure_host_pattern(A->stream);
    phif::LevelPlan h, d;
    h.grp = phif::classify_all(s);
    phif::build_level(s, h, phif::pattern_from_csr(h.grp, s.N, M.h_rowptr.get(), M.h_col.get()));
    phif::DevPlan0 dp;
    phif::plan_level0_device(s, M.rowptr.as<int64_t>(), M.col.as<int>(), M.nnz, d, dp, A->stream);
    phif::download_plan0(dp, d, A->stream);
    phif::compute_waves(d, d.grp.G);
    cudaStreamSynchronize(A->stream);
    auto cmp = [&](const char* name, const auto& a, const auto& b) {
      if (a.size() != b.size() || !std::equal(a.begin(), a.end(), b.begin())) {
        ++bad;
        rep += std::string(name) + " ";
      }
    };
    if (h.grp.G != d.grp.G) {
      ++bad;
      rep += "G ";
    }
    cmp("off", h.grp.off, d.grp.off);
    cmp("mem", h.grp.mem, d.grp.mem);
    cmp("kind", h.grp.kind, d.grp.kind);
    cmp("q", h.grp.q, d.grp.q);
    cmp("bits", h.grp.bits, d.grp.bits);
    cmp("bg", h.pat.bg, d.pat.bg);
    cmp("bh", h.pat.bh, d.pat.bh);
    cmp("adj_off", h.pat.adj_off, d.pat.adj_off);
    cmp("adj_nbr", h.pat.adj_nbr, d.pat.adj_nbr);
    cmp("adj_blk", h.pat.adj_blk, d.pat.adj_blk);
    cmp("boff", h.boff, d.boff);
    if (h.pool_doubles != d.pool_doubles) {
      ++bad;
      rep += "pool_doubles ";
    }
    cmp("interior", h.interior, d.interior);
    cmp("precond", h.precond, d.precond);
    cmp("skeleton", h.skeleton, d.skeleton);
    cmp("cell_nbr_off", h.cell_nbr_off, d.cell_nbr_off);
    cmp("cell_nbr", h.cell_nbr, d.cell_nbr);
    cmp("cell_nbr_blk", h.cell_nbr_blk, d.cell_nbr_blk);
    cmp("cell_nbr_col", h.cell_nbr_col, d.cell_nbr_col);
    cmp("cell_n", h.cell_n, d.cell_n);
    cmp("cell_b", h.cell_b, d.cell_b);
    cmp("tgt_blk", h.tgt_blk, d.tgt_blk);
    cmp("tgt_off", h.tgt_off, d.tgt_off);
    cmp("con_cell", h.con_cell, d.con_cell);
    cmp("con_row", h.con_row, d.con_row);
    cmp("con_col", h.con_col, d.con_col);
    cmp("scale_blk", h.scale_blk, d.scale_blk);
    cmp("sk_nbr_off", h.sk_nbr_off, d.sk_nbr_off);
    cmp("sk_nbr", h.sk_nbr, d.sk_nbr);
    cmp("sk_nbr_blk", h.sk_nbr_blk, d.sk_nbr_blk);
    cmp("sk_ndep", h.sk_ndep, d.sk_ndep);
    cmp("sk_succ_off", h.sk_succ_off, d.sk_succ_off);
    cmp("sk_succ", h.sk_succ, d.sk_succ);
    cmp("sk_wave", h.sk_wave, d.sk_wave);
    cmp("wave_off", h.wave_off, d.wave_off);
    cmp("wave_order", h.wave_order, d.wave_order);
    if (h.nwaves != d.nwaves) {
      ++bad;
      rep += "nwaves ";
    }
    rep += "| G=" + std::to_string(d.grp.G) + " blocks=" + std::to_string(d.pat.bg.size()) +
           " schur_contributions=" + std::to_string(d.con_cell.size());
  } catch (const std::exception& e) {
    rep = std::string("error: ") + e.what();
    bad = -1;
  }
  if (report && cap) {
    const size_t k = std::min(cap - 1, rep.size());
    std::memcpy(report, rep.data(), k);
    report[k] = 0;
  }
  return bad;
}

size_t phif_last_partial_stats(char* buf, size_t cap) {
  const std::string& s = g_partial_stats;
  if (buf && cap) {
    const size_t n = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return s.size();
}

int phif_num_levels(const phif_factor* F) { return (int)F->f->levels.size(); }

int phif_skeleton_sets(const phif_factor* F, int level, int64_t* counts, int32_t* rank, int32_t* nred,
                       int32_t* skel_dofs, int32_t* red_dofs) {
  const auto& lv = F->f->levels;
  if (level < 0 || level >= (int)lv.size()) return PHIF_ERROR;
  const phif::LevelRT& L = *lv[level];
  const phif::Groups& G = L.plan.grp;
  const int nsk = L.plan.root ? 0 : (int)L.plan.skeleton.size();
  int64_t rs = 0, ks = 0;
  for (int t = 0; t < nsk; ++t) {
    rs += L.h_rank[t];
    ks += G.size(L.plan.skeleton[t]) - L.h_rank[t];
  }
  counts[0] = nsk;
  counts[1] = rs;
  counts[2] = ks;
  if (!rank) return PHIF_OK;
  // the engine keeps S/R lists on device; recompute from the device copies
  std::vector<int> S(rs), R(ks);
  if (rs) cudaMemcpy(S.data(), L.s_S.p, rs * sizeof(int), cudaMemcpyDeviceToHost);
  if (ks) cudaMemcpy(R.data(), L.s_R.p, ks * sizeof(int), cudaMemcpyDeviceToHost);
  for (int t = 0; t < nsk; ++t) {
    rank[t] = L.h_rank[t];
    if (nred) nred[t] = G.size(L.plan.skeleton[t]) - L.h_rank[t];
  }
  if (skel_dofs) std::memcpy(skel_dofs, S.data(), rs * sizeof(int));
  if (red_dofs) std::memcpy(red_dofs, R.data(), ks * sizeof(int));
  return PHIF_OK;
}

int64_t phif_classify(int dim, int n, int m, int level, const int32_t* active, int64_t nactive, int32_t* group_of,
                      int32_t* kind_of_group, int64_t kind_cap) {
  try {
    phif::Spec s;
    s.init(dim, n, m);
    std::vector<int> act(active, active + nactive);
    phif::Groups g = phif::classify_set(s, level, act);
    std::vector<int> pos_of(s.N, -1);
    for (int64_t i = 0; i < nactive; ++i) pos_of[active[i]] = (int)i;
    for (int gi = 0; gi < g.G; ++gi)
      for (int64_t q = g.off[gi]; q < g.off[gi + 1]; ++q) group_of[pos_of[g.mem[q]]] = gi;
    if (kind_of_group)
      for (int gi = 0; gi < g.G && gi < kind_cap; ++gi) kind_of_group[gi] = g.kind[gi];
    return g.G;
  } catch (...) {
    return -1;
  }
}

size_t phif_plan_dryrun(int dim, int n, int m, const int64_t* rowptr, const int32_t* col, int keep, char* buf,
                        size_t cap) {
  std::string out;
  try {
    phif::Spec s;
    s.init(dim, n, m);
    std::vector<std::unique_ptr<phif::LevelPlan>> lv;
    std::vector<uint8_t> alive;
    out = "[";
    for (int l = 0; l <= s.L; ++l) {
      lv.push_back(std::make_unique<phif::LevelPlan>());
      phif::LevelPlan& P = *lv.back();
      auto t1 = std::chrono::steady_clock::now();
      std::vector<std::pair<int, int>> pairs;
      if (l == 0) {
        P.grp = phif::classify_all(s);
        auto tc = std::chrono::steady_clock::now();
        pairs = phif::pattern_from_csr(P.grp, s.N, rowptr, col);
        if (getenv("PHIF_DEBUG"))
          fprintf(stderr, "level 0: classify %.1f ms pattern %.1f ms\n",
                  std::chrono::duration<double, std::milli>(tc - t1).count(),
                  std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tc).count());
      } else {
        P.grp = phif::classify_next(s, lv[l - 1]->grp, alive);
        pairs = phif::pattern_next(*lv[l - 1], P.grp);
      }
      auto t2 = std::chrono::steady_clock::now();
      phif::build_level(s, P, std::move(pairs));
      auto t3 = std::chrono::steady_clock::now();
      if (getenv("PHIF_DEBUG"))
        fprintf(stderr, "level %d: classify+pattern %.1f ms build %.1f ms\n", l,
                std::chrono::duration<double, std::milli>(t2 - t1).count(),
                std::chrono::duration<double, std::milli>(t3 - t2).count());
      out += (l ? "," : "") + phif::level_json(P);
      alive.assign(P.grp.mem.size(), 0);
      for (int g = 0; g < P.grp.G; ++g) {
        if (P.grp.kind[g] == 0) continue;
        for (int64_t q = P.grp.off[g]; q < P.grp.off[g + 1]; ++q) {
          const int64_t pos = q - P.grp.off[g];
          alive[q] = (P.grp.kind[g] != 1 || keep < 0 || pos < keep) ? 1 : 0;
        }
      }
    }
    out += "]";
  } catch (const std::exception& e) {
    out = std::string("{\"error\":\"") + e.what() + "\"}";
  }
  if (buf && cap) {
    const size_t k = std::min(cap - 1, out.size());
    std::memcpy(buf, out.data(), k);
    buf[k] = 0;
  }
  return out.size();
}

}  // extern "C"
