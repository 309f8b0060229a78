"""Debug driver: GPU path vs oracle on small problems (prints per-case summary)."""
import sys, time, json, traceback
import numpy as np
sys.path.insert(0, ".")
from paper_1808_01364_b200 import GridSpec, generate_field, assemble_operator, baseline_problem
from paper_1808_01364_b200 import factorization as gf, krylov as gk, diagnostics as gd
from oracle import phif as of, krylov as ok, diagnostics as od

cases = [(2, 16, 4, "exact", 0.0), (2, 32, 4, "phif", 1e-6), (2, 32, 8, "hif", 1e-6), (3, 16, 4, "exact", 0.0),
         (3, 16, 4, "phif", 1e-3), ("c1",), ("c4", 32)]
if len(sys.argv) > 1:
    cases = [eval(a) for a in sys.argv[1:]]
for case in cases:
    try:
        if isinstance(case[0], str):
            from paper_1808_01364_b200.grid import CONFIGS
            cfg = CONFIGS[case[0]]
            spec, A, _ = baseline_problem(case[0], 0, case[1] if len(case) > 1 else None)
            method, eps = cfg.method, cfg.eps[0]
        else:
            dim, n, m, method, eps = case
            spec = GridSpec(dim, n, m)
            A = assemble_operator(generate_field(spec, 1), 0.0)
        t = time.time(); Fg = gf.factorize(A, spec, eps, method, timing=True); tg = time.time() - t
        t = time.time(); Fo = of.factorize(A, spec, eps, method); to = time.time() - t
        # skeleton sets
        mism = 0; tot = 0
        for lev in range(spec.levels):
            gs = Fg.skeleton_sets(lev)
            os_ = [(r.skeleton, r.redundant) for r in Fo.levels[lev].skeletonize]
            # oracle only records groups with redundant dofs; compare redundant sets keyed by group
            ored = {tuple(np.sort(r.redundant)) for r in Fo.levels[lev].skeletonize}
            gred = {tuple(np.sort(r)) for (s, r) in gs if len(r)}
            tot += len(ored | gred); mism += len(ored ^ gred)
        rng = np.random.default_rng(0)
        b = rng.standard_normal((A.n, 3))
        yg = gf.apply_inverse(Fg, b); yo = of.apply_inverse(Fo, b)
        dinv = np.linalg.norm(yg - yo) / np.linalg.norm(yo)
        x = rng.standard_normal(A.n)
        einv = np.linalg.norm(gf.apply_inverse(Fg, A.csr @ x) - x) / np.linalg.norm(x)
        bb = rng.standard_normal(A.n)
        xg, rg = gk.pcg(A, bb, precond=Fg, tol=1e-12)
        xo, ro = ok.pcg(A, bb, precond=Fo, tol=1e-12)
        dx = np.linalg.norm(xg - xo) / np.linalg.norm(xo)
        esg = gd.estimate_solve_error(A, Fg); eso = od.estimate_solve_error(A, Fo)
        print(json.dumps(dict(case=str(case), N=A.n, SL_gpu=Fg.SL, SL_oracle=Fo.SL, skel_mismatch=f"{mism}/{tot}",
                              apply_inv_reldiff=dinv, inv_err=einv, ni_gpu=rg.n_i, ni_oracle=ro.n_i, x_reldiff=dx,
                              es_gpu=esg.value, es_oracle=eso.value, t_gpu=round(tg, 3), t_oracle=round(to, 3))))
        st = Fg.stats
        print("  stats:", json.dumps({k: v for k, v in st.items() if k != "levels"}))
        for lv in st["levels"]:
            print("   ", json.dumps(lv))
    except Exception:
        print("CASE FAILED", case)
        traceback.print_exc()
    sys.stdout.flush()
