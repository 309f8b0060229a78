"""Full-size oracle fixtures for the -m gpu parity tests at the BASELINE sizes.

Runs the CPU oracle (oracle/, which restates SPEC.md:229-453 on the reference's own primitives)
on a BASELINE config at its full size with the seeded inputs of paper_1808_01364_b200.grid, and
writes tests/golden/fullsize_<tag>.npz:

* the input checksum (sha256 of the CSR arrays), so the GPU box proves it rebuilt the same A;
* the outcome: "ok", or "not-spd" with (level, stage, group, pivot) of the NotSpdError;
* when it factorizes: |S_L|, per level the rank and the sorted redundant DOFs of every
  separator (classify order), PCG n_i / relres for the config's right-hand sides, the solution
  on a seeded subset of 4096 DOFs and its projection on 64 seeded Gaussian vectors (a
  norm-preserving sketch: |S d| / |S x| estimates |d| / |x| within ~25% at 64 rows), e_s;
* the oracle's per-level stage times on this host (cores / model recorded).

Usage (in the build container, where the oracle's time is free):
    python tests/golden/make_fullsize.py c5 1e-2 phif
    python tests/golden/make_fullsize.py c3 1e-4 phif
"""
import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import diagnostics as odiag  # noqa: E402
from oracle import krylov as okry  # noqa: E402
from oracle import phif as ophif  # noqa: E402
from oracle.errors import NotSpdError  # noqa: E402
from paper_1808_01364_b200.grid import CONFIGS, baseline_problem, baseline_rhs  # noqa: E402

SKETCH_ROWS = 64
SUBSET = 4096


def csr_sha(A):
    h = hashlib.sha256()
    for a in (A.csr.indptr.astype(np.int64), A.csr.indices.astype(np.int32), A.csr.data.astype(np.float64)):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def sketch(X, N, seed):
    """64 x nrhs projection of X on seeded Gaussian rows, streamed in row blocks (memory-bounded)."""
    rng = np.random.default_rng([seed, 99])
    out = np.zeros((SKETCH_ROWS, X.shape[1]))
    for r0 in range(0, SKETCH_ROWS, 8):
        S = rng.standard_normal((8, N))
        out[r0:r0 + 8] = S @ X
    return out


def subset_index(N, seed):
    return np.sort(np.random.default_rng([seed, 98]).choice(N, size=min(SUBSET, N), replace=False))


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def _progress():
    """Print every oracle stage as it finishes (the full-size runs take tens of minutes)."""
    t_start = time.perf_counter()
    for name in ("eliminate_cells", "precondition_blocks", "skeletonize_separators"):
        fn = getattr(ophif, name)

        def wrap(*a, _fn=fn, _name=name, **k):
            t0 = time.perf_counter()
            out = _fn(*a, **k)
            li = 3 if _name == "skeletonize_separators" else 2
            lev = k.get("level", a[li] if len(a) > li else None)
            print(f"  [{time.perf_counter() - t_start:8.1f} s] level {lev} {_name} {time.perf_counter() - t0:.1f} s",
                  flush=True)
            return out
        setattr(ophif, name, wrap)


def main():
    name, eps, method = sys.argv[1], float(sys.argv[2]), sys.argv[3]
    nrhs = int(sys.argv[4]) if len(sys.argv) > 4 else None
    seed = 0
    cfg = CONFIGS[name]
    tag = f"{name}_{method}_{eps:g}"
    out = os.path.join(ROOT, "tests", "golden", f"fullsize_{tag}.npz")
    t0 = time.perf_counter()
    spec, A, _ = baseline_problem(name, seed, None)
    meta = {"config": name, "eps": eps, "method": method, "seed": seed, "N": int(A.n), "nnz": int(A.nnz),
            "csr_sha256": csr_sha(A), "t_problem_s": time.perf_counter() - t0, "host_cores": os.cpu_count(),
            "cpu_model": cpu_model(), "omp_threads": os.environ.get("OPENBLAS_NUM_THREADS", "all"),
            "generator": "tests/golden/make_fullsize.py"}
    print(json.dumps(meta), flush=True)
    arrays = {}
    _progress()
    t0 = time.perf_counter()
    try:
        F = ophif.factorize(A, spec, eps, method)
    except NotSpdError as e:
        meta.update(outcome="not-spd", level=e.level, stage=e.stage, group=e.group, pivot=e.pivot,
                    t_factor_s=time.perf_counter() - t0)
        print(json.dumps(meta), flush=True)
        np.savez_compressed(out, meta=json.dumps(meta))
        return
    meta.update(outcome="ok", t_factor_s=time.perf_counter() - t0, SL=int(F.SL), levels=F.stats["levels"])
    print(json.dumps(meta), flush=True)
    for lev, lv in enumerate(F.levels):
        recs = lv.skeletonize
        arrays[f"l{lev}_group"] = np.array([r.group for r in recs], dtype=np.int32)
        arrays[f"l{lev}_nred"] = np.array([len(r.redundant) for r in recs], dtype=np.int32)
        arrays[f"l{lev}_red"] = (np.concatenate([np.sort(r.redundant) for r in recs]).astype(np.int32)
                                 if recs else np.zeros(0, np.int32))
    meta["nlevels"] = len(F.levels)
    k = nrhs or cfg.nrhs
    B = baseline_rhs(cfg, A.n, seed, k)
    t0 = time.perf_counter()
    X, rep = okry.pcg(A, B, precond=F, tol=cfg.tol)
    meta["t_pcg_s"] = time.perf_counter() - t0
    arrays["n_i"] = np.atleast_1d(rep.n_i).astype(np.int32)
    arrays["relres"] = np.atleast_1d(rep.relres).astype(np.float64)
    idx = subset_index(A.n, seed)
    arrays["x_idx"] = idx.astype(np.int64)
    arrays["x_sub"] = X[idx]
    arrays["x_sketch"] = sketch(X, A.n, seed)
    arrays["x_norm"] = np.linalg.norm(X, axis=0)
    print(json.dumps({"n_i": arrays["n_i"].tolist(), "t_pcg_s": meta["t_pcg_s"]}), flush=True)
    del X
    t0 = time.perf_counter()
    es = odiag.estimate_solve_error(A, F)
    meta.update(e_s=es.value, e_s_iters=es.iterations, e_s_converged=bool(es.converged),
                t_es_s=time.perf_counter() - t0)
    print(json.dumps({"e_s": es.value, "iters": es.iterations, "t_es_s": meta["t_es_s"]}), flush=True)
    np.savez_compressed(out, meta=json.dumps(meta), **arrays)
    print("wrote", out, flush=True)


if __name__ == "__main__":
    main()
