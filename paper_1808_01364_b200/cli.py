"""bench_cli of the drop-in: the reference's command-line harness over the B200 path.

    python -m paper_1808_01364_b200.cli <gen|factor|solve|bench|scaling> [flags]

Global flags: --dim {2,3} --n --m (8) --eps --method {hif,phif,exact} --seed
--contrast (1e4) --tol (1e-12) --maxit (500) --out --seeds (count); plus --config c1..c5 to take
the problem from a BASELINE.json configuration (its field recipe, b, m, n and eps) and --eps-list /
--methods / --n-list for sweeps. Exit codes: 0 ok, 2 NotSpd (reported as data, never a crash),
1 other errors, 64 usage (unknown flags).

`bench` runs, for every (method, eps, n, seed): generate the field, assemble, factorize (NotSpd ->
status not-spd), estimate e_a and e_s, solve one N(0,1) right-hand side by PCG to --tol, and
appends one row per run to the CSV as soon as it is measured (partial runs persist). The header is
exactly SPEC.md:510's:

    method,eps,dim,n,N,seed,SL,e_a,e_s,n_i,t_factor_s,t_apply_s,mem_bytes,status

`scaling` reads such CSVs and emits (N, method, factor_time, apply_time, memory) plus the fitted
log-log slope of each series; fewer than two sizes is refused.
"""

from __future__ import annotations

import argparse
import csv
import json
import os
import sys
import time

import numpy as np

CSV_HEADER = ["method", "eps", "dim", "n", "N", "seed", "SL", "e_a", "e_s", "n_i", "t_factor_s", "t_apply_s",
              "mem_bytes", "status"]
EXIT_OK, EXIT_ERROR, EXIT_NOT_SPD, EXIT_USAGE = 0, 1, 2, 64


class _Parser(argparse.ArgumentParser):
    def error(self, message):   # usage errors exit 64, not argparse's 2 (= NotSpd here)
        self.print_usage(sys.stderr)
        sys.stderr.write(f"{self.prog}: error: {message}\n")
        raise SystemExit(EXIT_USAGE)


def _floats(s):
    return [float(v) for v in s.split(",") if v]


def _ints(s):
    return [int(v) for v in s.split(",") if v]


def build_parser():
    p = _Parser(prog="hifsolve-b200", description=__doc__.splitlines()[0])
    p.add_argument("command", choices=["gen", "factor", "solve", "bench", "scaling"])
    p.add_argument("--dim", type=int, choices=[2, 3], default=2)
    p.add_argument("--n", type=int, default=None)
    p.add_argument("--m", type=int, default=8)
    p.add_argument("--eps", type=float, default=1e-6)
    p.add_argument("--method", choices=["hif", "phif", "exact"], default="phif")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--contrast", type=float, default=1e4)
    p.add_argument("--tol", type=float, default=1e-12)
    p.add_argument("--maxit", type=int, default=500)
    p.add_argument("--out", default=None)
    p.add_argument("--seeds", type=int, default=1)
    p.add_argument("--config", choices=["c1", "c2", "c3", "c3p", "c4", "c5"], default=None)
    p.add_argument("--eps-list", type=_floats, default=None)
    p.add_argument("--n-list", type=_ints, default=None)
    p.add_argument("--methods", default=None, help="comma list, e.g. hif,phif")
    p.add_argument("--no-estimates", action="store_true", help="skip e_a / e_s (large runs)")
    p.add_argument("inputs", nargs="*", help="CSV files (scaling)")
    return p


def _problem(args, n, seed):
    from .grid import GridSpec, assemble_operator, baseline_problem, generate_field
    if args.config:
        spec, A, field = baseline_problem(args.config, seed, n)
        return spec, A, field
    spec = GridSpec(args.dim, n if n is not None else 128, args.m)
    field = generate_field(spec, seed, args.contrast)
    return spec, assemble_operator(field), field


def run_one(args, method, eps, n, seed, estimates=True):
    """One BenchRow as a dict in CSV_HEADER order."""
    from . import diagnostics, factorization, krylov
    from .errors import NotSpdError
    spec, A, _ = _problem(args, n, seed)
    row = {"method": method, "eps": eps if method != "exact" else 0.0, "dim": spec.dim, "n": spec.n,
           "N": spec.ndofs, "seed": seed, "SL": "", "e_a": "", "e_s": "", "n_i": "", "t_factor_s": "",
           "t_apply_s": "", "mem_bytes": "", "status": "ok"}
    factorization.device_matrix(A)
    t0 = time.perf_counter()
    try:
        F = factorization.factorize(A, spec, eps, method)
    except NotSpdError as e:
        row["t_factor_s"] = time.perf_counter() - t0
        row["status"] = "not-spd"
        row["_notspd"] = {"level": e.level, "stage": e.stage, "group": e.group, "pivot": e.pivot}
        return row
    row["t_factor_s"] = time.perf_counter() - t0
    st = F.stats
    row["SL"] = st["SL"]
    row["mem_bytes"] = st["mem_bytes"]
    b = np.random.default_rng([seed, 1]).standard_normal(spec.ndofs)
    t0 = time.perf_counter()
    factorization.apply_inverse(F, b)
    row["t_apply_s"] = time.perf_counter() - t0
    if estimates:
        row["e_a"] = diagnostics.estimate_apply_error(A, F).value
        row["e_s"] = diagnostics.estimate_solve_error(A, F).value
    x, rep = krylov.pcg(A, b, precond=F, tol=args.tol, maxit=args.maxit)
    row["n_i"] = rep.n_i
    if not rep.converged:
        row["status"] = "maxit"
    return row


def _append_csv(path, row):
    new = not os.path.exists(path) or os.path.getsize(path) == 0
    with open(path, "a", newline="") as fh:
        w = csv.writer(fh)
        if new:
            w.writerow(CSV_HEADER)
        w.writerow([row[k] for k in CSV_HEADER])


def fit_slope(xs, ys):
    """Least-squares slope of log(y) against log(x)."""
    lx, ly = np.log(np.asarray(xs, float)), np.log(np.asarray(ys, float))
    return float(np.polyfit(lx, ly, 1)[0])


def emit_scaling(rows):
    """Per (method) series over N: factor/apply time and memory, with log-log slopes."""
    series = {}
    for r in rows:
        if r.get("status", "ok") != "ok":
            continue
        series.setdefault(r["method"], []).append(r)
    out = {"rows": [], "slopes": {}}
    for method, rs in sorted(series.items()):
        by_n = {}
        for r in rs:
            by_n.setdefault(int(r["N"]), []).append(r)
        Ns = sorted(by_n)
        if len(Ns) < 2:
            raise ValueError(f"scaling needs at least two sizes (method {method} has {len(Ns)})")
        agg = []
        for N in Ns:
            g = by_n[N]
            agg.append((N, float(np.median([float(r["t_factor_s"]) for r in g])),
                        float(np.median([float(r["t_apply_s"]) for r in g])),
                        float(np.median([float(r["mem_bytes"]) for r in g]))))
            out["rows"].append({"N": N, "method": method, "factor_time": agg[-1][1], "apply_time": agg[-1][2],
                                "memory": agg[-1][3]})
        out["slopes"][method] = {"factor_time": fit_slope([a[0] for a in agg], [a[1] for a in agg]),
                                 "apply_time": fit_slope([a[0] for a in agg], [a[2] for a in agg]),
                                 "memory": fit_slope([a[0] for a in agg], [a[3] for a in agg])}
    return out


def main(argv=None):
    args = build_parser().parse_args(argv)
    try:
        if args.command == "scaling":
            rows = []
            for path in args.inputs:
                with open(path) as fh:
                    rows.extend(csv.DictReader(fh))
            res = emit_scaling(rows)
            text = json.dumps(res, indent=1)
            if args.out:
                with open(args.out, "w") as fh:
                    fh.write(text + "\n")
            print(text)
            return EXIT_OK
        if args.command == "gen":
            spec, A, field = _problem(args, args.n, args.seed)
            if args.out:
                A.write_coordinate(args.out)   # MatrixMarket coordinate, lower triangle
            print(json.dumps({"dim": spec.dim, "n": spec.n, "m": spec.m, "N": spec.ndofs, "nnz": int(A.nnz),
                              "seed": args.seed, "generator": "numpy-pcg64"}))
            return EXIT_OK
        methods = args.methods.split(",") if args.methods else [args.method]
        eps_list = args.eps_list or [args.eps]
        n_list = args.n_list or [args.n]
        if args.command in ("factor", "solve"):
            row = run_one(args, methods[0], eps_list[0], n_list[0], args.seed,
                          estimates=args.command == "solve" and not args.no_estimates)
            print(json.dumps({k: v for k, v in row.items()}))
            return EXIT_NOT_SPD if row["status"] == "not-spd" else EXIT_OK
        # bench
        out = args.out or "bench.csv"
        any_notspd = False
        for method in methods:
            for eps in eps_list:
                for n in n_list:
                    for seed in range(args.seed, args.seed + args.seeds):
                        row = run_one(args, method, eps, n, seed, estimates=not args.no_estimates)
                        _append_csv(out, row)
                        any_notspd |= row["status"] == "not-spd"
                        print(json.dumps({k: row[k] for k in CSV_HEADER}), flush=True)
        return EXIT_OK
    except SystemExit:
        raise
    except Exception as e:   # configuration / engine errors
        from .errors import NotSpdError
        if isinstance(e, NotSpdError):
            return EXIT_NOT_SPD
        sys.stderr.write(f"error: {e}\n")
        return EXIT_ERROR


if __name__ == "__main__":
    sys.exit(main())
