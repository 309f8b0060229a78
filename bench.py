#!/usr/bin/env python
"""Benchmark of the B200 PHIF factorize / PCG path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--workload c5]

A "step" is one factorization of the workload's matrix (inputs resident in HBM);
`value` = factorization DOF/s summed over ranks (replicas, weak scaling: every rank
factors its own seeded problem; max-over-ranks device time). The PCG solve of the
config's right-hand sides (solve ms/RHS, n_i) is measured after the factor steps.
`e2e` repeats the factorization through the public C-ABI with HOST CSR buffers
(upload inside the timed region, statistics read back). `roofline` is the
dominant (level, stage) launch of a timed step: algorithmic flops (SURVEY.md 8(d)
counts) / its CUDA-event duration on the launch stream, against the measured FP64
cuBLAS DGEMM peak (profiles/fp64_peak_r01.json) or the measured HBM copy peak.
`--impl reference` times the CPU oracle (the reference ships no factorization
module, so the restated path in oracle/ is the reference arm) on a bounded sample.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1808_01364_b200.grid import CONFIGS, baseline_problem, baseline_rhs  # noqa: E402

WORKLOADS = {
    # name: config, eps, grid n (None = full size), CPU sample n
    "c5": ("c5", 1e-2, None, 64),
    "c4": ("c4", 1e-3, None, 32),
    "c2": ("c2", 1e-3, None, 256),
    "c3p": ("c3p", 1e-4, None, 512),
    "c1": ("c1", 1e-6, None, 128),
}
FP64_PEAK_TFLOPS = 35.47     # measured cuBLAS DGEMM 8192^3 on this pool (profiles/fp64_peak_r01.json)


def load_peaks():
    hbm = 6540.2
    try:
        hbm = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        pass
    fp64 = FP64_PEAK_TFLOPS
    try:
        fp64 = float(json.load(open(os.path.join(ROOT, "profiles", "fp64_peak_r01.json")))["dgemm_8192_tflops"])
    except Exception:
        pass
    return hbm, fp64


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = "gloo" if args.impl == "reference" else "nccl"
        if backend == "nccl":
            import torch
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
        pg = dist
    return world, rank, local, pg


def reduce_max_sum(pg, tmax, units, device=None):
    """Max of the timed duration and sum of processed units over ranks (replica timing)."""
    if pg is None:
        return tmax, units
    import torch
    t = torch.tensor([tmax], dtype=torch.float64, device=device)
    u = torch.tensor([units], dtype=torch.float64, device=device)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    pg.all_reduce(u, op=pg.ReduceOp.SUM)
    return float(t.item()), float(u.item())


def cpu_sample(workload, seed=0):
    """Bounded CPU sample: the oracle factorization of the workload's recipe on a smaller grid."""
    from oracle import phif as ophif
    cfg, eps, _, sn = WORKLOADS[workload]
    spec, A, _ = baseline_problem(cfg, seed, sn)
    t0 = time.perf_counter()
    F = ophif.factorize(A, spec, eps, CONFIGS[cfg].method)
    dt = time.perf_counter() - t0
    return A.n / dt, dt, spec, F


def _fullsize_note(workload):
    full = cpu_fullsize(workload)
    if not full:
        return None
    return {"value": full["dofs_per_s"], "unit": "DOF/s", "N": full["N"], "seconds": full["t_factor_s"],
            "cores": full["cores"], "cpu_model": full["cpu_model"],
            "source": f"profiles/cpu_fullsize_{workload}_r02.json (the oracle's full-size factorization timed on "
                      f"the GPU box host; too long to repeat per step)"}


def run_reference(args, world, rank, pg):
    if rank != 0:
        return
    cfg, eps, n, sn = WORKLOADS[args.workload]
    for _ in range(args.warmup):
        cpu_sample(args.workload)
    times, N = [], 0
    for _ in range(args.steps):
        dofs, dt, spec, F = cpu_sample(args.workload)
        times.append(dt)
        N = spec.ndofs
    t = float(np.sum(times))
    val = N * args.steps / t
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "DOF/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE recipe, numpy-pcg64)",
            "config": {"workload": args.workload, "cfg": CONFIGS[cfg].description, "eps": eps,
                       "sample_grid_n": sn, "sample_N": N},
            "cpu_baseline": {"value": val, "unit": "DOF/s", "cores": os.cpu_count(), "kind": "port",
                             "sample": f"oracle factorize of the {cfg} recipe on a {sn}-grid (N={N}), "
                                       f"numpy/scipy OpenBLAS with all host threads"},
            "fullsize": _fullsize_note(args.workload),
            "e2e": {"value": val, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# BASELINE.json metric (both arms report it under the same name)
METRIC = "factor DOF/s (HIF factor DOF/s & FP64 roofline fraction; PCG iters; solve ms/RHS)"


def dominant_stage(stats):
    """The longest (level, stage) of the step, whatever bounds it."""
    names = ["repack", "eliminate", "precondition", "id", "skel_update"]
    keys = ["t_repack_ms", "t_eliminate_ms", "t_precondition_ms", "t_id_ms", "t_skel_update_ms"]
    best = None
    for lv in stats["levels"]:
        for si, key in enumerate(keys):
            t = lv.get(key, 0.0)
            if best is None or t > best[0]:
                best = (t, lv["level"], names[si])
    return {"level": best[1], "stage": best[2], "t_ms": best[0]}


def dominant_roofline(stats, hbm_peak, fp64_peak):
    """Roofline of the dominant batched dense stage: the longest (level, stage) among the
    DMMA-batched stages (eliminate / precondition / skeleton update, the root). The ID stages are
    excluded: their cost is the sequential dlaqp2 pivot chain, latency-bound by construction
    (no roofline for the pivot search); they are reported under
    `dominant_stage` and in `roofline_levels` with their achieved rates."""
    names = ["repack", "eliminate", "precondition", "id", "skel_update"]
    keys = ["t_repack_ms", "t_eliminate_ms", "t_precondition_ms", "t_id_ms", "t_skel_update_ms"]
    best = None
    for lv in stats["levels"]:
        for si, key in enumerate(keys):
            if names[si] in ("repack", "id"):
                continue
            t = lv.get(key, 0.0)
            if best is None or t > best[0]:
                best = (t, lv["level"], si, lv["flops"][si], lv["bytes"][si])
    t_ms, lev, si, fl, by = best
    intensity = fl / by if by else 0.0
    # measured DRAM traffic per launch of the stage's kernel (ncu --set full, committed profile)
    traffic, tnote = None, None
    try:
        pdir = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles")
        tpath = os.path.join(pdir, "traffic_r02.json")
        tj = json.load(open(tpath if os.path.exists(tpath) else os.path.join(pdir, "traffic_r01.json")))
        ent = tj.get(f"level {lev} {names[si]}")
        if ent:
            traffic = ent["dram_bytes_per_launch"]
            tnote = f"dram bytes per {ent['kernel']} launch, {ent['source']}"
    except (OSError, ValueError, KeyError):
        pass
    ridge = fp64_peak * 1e12 / (hbm_peak * 1e9)
    if intensity >= ridge:
        ach = fl / (t_ms * 1e-3) / 1e12
        return {"bound": "tensor", "achieved": ach, "peak": fp64_peak, "unit": "TFLOP/s", "frac": ach / fp64_peak,
                "traffic": traffic, "traffic_note": tnote, "kernel": f"level {lev} {names[si]}", "time_ms": t_ms,
                "algorithmic_flops": fl,
                "algorithmic_bytes": by, "peak_source": "measured cuBLAS DGEMM (profiles/fp64_peak_r01.json)"}
    ach = by / (t_ms * 1e-3) / 1e9
    return {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
            "traffic": traffic, "traffic_note": tnote, "kernel": f"level {lev} {names[si]}", "time_ms": t_ms,
            "algorithmic_flops": fl,
            "algorithmic_bytes": by, "peak_source": "MEASURED_PEAKS.json hbm_gbs"}


STAGES = ["repack", "eliminate", "precondition", "id", "skel_update"]
STAGE_KEYS = ["t_repack_ms", "t_eliminate_ms", "t_precondition_ms", "t_id_ms", "t_skel_update_ms"]


def roofline_levels(stats, hbm_peak, fp64_peak):
    """Per (level, stage): algorithmic flops and bytes (SURVEY.md 8(d) counts accumulated by the
    engine from the actual shapes) over the stage's CUDA-event time on the launch stream, as
    fractions of the measured FP64 (DGEMM) and HBM (copy) peaks. `bound` is the roofline the
    stage's arithmetic intensity puts it under (ridge = fp64_peak / hbm_peak)."""
    ridge = fp64_peak * 1e12 / (hbm_peak * 1e9)
    out = []
    for lv in stats["levels"]:
        for si, key in enumerate(STAGE_KEYS):
            t = float(lv.get(key, 0.0))
            fl, by = float(lv["flops"][si]), float(lv["bytes"][si])
            if t <= 0.0 or (fl == 0.0 and by == 0.0):
                continue
            tf = fl / (t * 1e-3) / 1e12
            gb = by / (t * 1e-3) / 1e9
            root = lv["level"] == stats["levels"][-1]["level"] and si == 1
            out.append({"level": lv["level"], "stage": "root" if root else STAGES[si], "t_ms": round(t, 4), "flops": fl, "bytes": by,
                        "tflops": round(tf, 3), "gbs": round(gb, 1), "frac_fp64": round(tf / fp64_peak, 4),
                        "frac_hbm": round(gb / hbm_peak, 4),
                        "bound": "tensor" if by and fl / by >= ridge else "hbm"})
    return out


def cpu_fullsize(workload):
    """Committed full-size CPU-oracle timing of the workload, measured on the GPU box host
    (profiles/cpu_fullsize_<workload>_r02.json, written by tools/cpu_fullsize.py)."""
    path = os.path.join(ROOT, "profiles", f"cpu_fullsize_{workload}_r02.json")
    try:
        return json.load(open(path))
    except (OSError, ValueError):
        return None


def run_b200(args, world, rank, local, pg):
    import torch

    from paper_1808_01364_b200 import _lib, factorization, krylov

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev).cuda_stream
    cfg_name, eps, n, sn = WORKLOADS[args.workload]
    cfg = CONFIGS[cfg_name]
    spec, A, _ = baseline_problem(cfg_name, rank, n)
    N = spec.ndofs
    dm = factorization.device_matrix(A, stream)
    L = _lib.lib()

    def sync():
        torch.cuda.synchronize(dev)
        if pg is not None:
            pg.barrier()

    F = None
    for _ in range(args.warmup):
        F = None
        F = factorization.factorize(dm, spec, eps, cfg.method, stream=stream, timing=True)
    sync()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    launches0 = L.phif_launch_count()
    with ClockSampler(local) as clocks:
        ev0.record()
        for _ in range(args.steps):
            F = None
            F = factorization.factorize(dm, spec, eps, cfg.method, stream=stream, timing=True)
        ev1.record()
        torch.cuda.synchronize(dev)
    launches = L.phif_launch_count() - launches0
    t_factor = ev0.elapsed_time(ev1) * 1e-3
    t_all, units = reduce_max_sum(pg, t_factor, float(N * args.steps), dev if pg else None)
    value = units / t_all
    stats = F.stats
    hbm_peak, fp64_peak = load_peaks()
    roof = dominant_roofline(stats, hbm_peak, fp64_peak)

    # PCG solve with the config's right-hand sides (device-resident inputs)
    B = baseline_rhs(cfg, N, rank)
    Bd = torch.from_numpy(B).to(dev)
    Xd = torch.zeros_like(Bd)
    import ctypes as C
    iters = np.zeros(B.shape[1], dtype=np.int32)
    relres = np.zeros(B.shape[1])
    conv = np.zeros(B.shape[1], dtype=np.int32)
    err = _lib.phif_error()
    # untimed warm-up solve (apply workspaces for this nrhs are allocated on the first call)
    rc = L.phif_pcg(dm.handle, F.handle, C.c_void_p(Bd.data_ptr()), C.c_void_p(Xd.data_ptr()), B.shape[1],
                    cfg.tol, 2, C.c_void_p(stream), _lib.ptr(iters), _lib.ptr(relres), _lib.ptr(conv),
                    None, None, C.byref(err))
    _lib.raise_for(rc, err)
    Xd.zero_()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    rc = L.phif_pcg(dm.handle, F.handle, C.c_void_p(Bd.data_ptr()), C.c_void_p(Xd.data_ptr()), B.shape[1],
                    cfg.tol, 500, C.c_void_p(stream), _lib.ptr(iters), _lib.ptr(relres), _lib.ptr(conv),
                    None, None, C.byref(err))
    e1.record()
    torch.cuda.synchronize(dev)
    _lib.raise_for(rc, err)
    t_solve = e0.elapsed_time(e1)

    # e_s = ||I - G^-1 A G^-T|| (power iteration on the device)
    from paper_1808_01364_b200 import diagnostics
    t0 = time.perf_counter()
    es = diagnostics.estimate_solve_error(A, F)
    t_es = time.perf_counter() - t0

    # e2e: public API with host buffers (CSR upload + factorize + stats read-back)
    h2d = A.csr.indptr.size * 8 + A.csr.indices.size * 4 + A.csr.data.size * 8
    e2e_steps = max(1, min(args.steps, 3))
    for it in range(1 + e2e_steps):   # one untimed warm-up (allocator growth), then timed steps
        if it == 1:
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
        A._device = None
        F2 = factorization.factorize(A, spec, eps, cfg.method, stream=stream)
        _ = F2.stats["SL"]
        F2 = None
    torch.cuda.synchronize(dev)
    t_e2e = (time.perf_counter() - t0) / e2e_steps
    t_e2e_all, u_e2e = reduce_max_sum(pg, t_e2e, float(N), dev if pg else None)
    stats_len = len(json.dumps(stats))
    # e2e through on-device generation: host RNG draw of the field's white
    # noise, upload of that one lattice, smoothing + threshold + assembly on the device, factorize
    gen = None
    if cfg.recipe.startswith("thresh_"):
        from paper_1808_01364_b200.device_problem import device_baseline_problem
        for it in range(1 + e2e_steps):
            if it == 1:
                torch.cuda.synchronize(dev)
                t0 = time.perf_counter()
            _, M = device_baseline_problem(cfg_name, rank, n, stream=stream)
            F3 = factorization.factorize(M, spec, eps, cfg.method, stream=stream)
            _ = F3.stats["SL"]
            F3 = None
            gen_h2d = M.h2d_bytes
            M = None
        torch.cuda.synchronize(dev)
        t_gen = (time.perf_counter() - t0) / e2e_steps
        gen = {"value": N / t_gen, "unit": "DOF/s", "h2d_bytes_per_step": int(gen_h2d),
               "d2h_bytes_per_step": int(stats_len),
               "path": "host numpy draw of the white noise + device Gaussian filter, threshold and stencil assembly "
                       "(bit-identical to the host recipe) + factorize"}
    # e2e solve with host right-hand sides (H2D of B, D2H of X inside the call); one untimed
    # one-iteration warm-up call first (the pinned staging areas are allocated by the first host call)
    krylov.pcg(A, B, precond=F, tol=cfg.tol, maxit=1, stream=stream)
    t0 = time.perf_counter()
    Xh, rep = krylov.pcg(A, B, precond=F, tol=cfg.tol, stream=stream)
    t_e2e_solve = time.perf_counter() - t0

    if rank != 0:
        return
    cpu = None
    if world == 1 and not args.no_cpu:
        dofs, dt, sspec, _ = cpu_sample(args.workload)
        sampled = {"value": dofs, "unit": "DOF/s", "cores": os.cpu_count(), "N": sspec.ndofs, "seconds": dt,
                   "sample": f"oracle factorize of the {cfg_name} recipe on a {sn}-grid (N={sspec.ndofs}), "
                             f"timed live in this run; numpy/scipy OpenBLAS using all host threads"}
        full = cpu_fullsize(args.workload)
        if full and full.get("N") == N:
            cpu = {"value": full["dofs_per_s"], "unit": "DOF/s", "cores": full["cores"], "kind": "port",
                   "N": N, "seconds": full["t_factor_s"],
                   "sample": f"full-size oracle factorization of {cfg_name} (N={N}) on the GPU box host "
                             f"({full['cpu_model']}, {full['cores']} cores), committed in "
                             f"profiles/cpu_fullsize_{args.workload}_r02.json; the live bounded sample of this "
                             f"run is under 'sampled'",
                   "sampled": sampled}
        else:
            cpu = dict(sampled, kind="port")
    line = {
        "metric": METRIC,
        "value": value, "unit": "DOF/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t_all / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded BASELINE recipe, numpy-pcg64)",
        "config": {"workload": args.workload, "cfg": cfg.description, "N": N, "eps": eps, "method": cfg.method,
                   "nrhs": int(B.shape[1]), "parallelism": f"replicas x{world}",
                   "l2": "inputs larger than L2 (factor records %.1f GB per step)" % (stats["mem_bytes"] / 1e9)},
        "SL": stats["SL"], "pcg_iters": [int(v) for v in iters], "pcg_relres_max": float(np.max(relres)),
        "solve_ms_per_rhs": t_solve / B.shape[1], "t_factor_ms": 1e3 * t_all / args.steps,
        "t_plan_ms": stats["t_plan_ms"],
        "e2e": {"value": u_e2e / t_e2e_all, "unit": "DOF/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(stats_len),
                "solve_ms_per_rhs": 1e3 * t_e2e_solve / B.shape[1],
                "solve_h2d_bytes": int(B.nbytes), "solve_d2h_bytes": int(Xh.nbytes),
                "generated_on_device": gen},
        "roofline": roof,
        "dominant_stage": dict(dominant_stage(stats), note="the ID stages are the sequential pivot chain "
                               "(latency-bound); their achieved FP64/HBM fractions are in roofline_levels"),
        "roofline_levels": roofline_levels(stats, hbm_peak, fp64_peak),
        "e_s": es.value, "e_s_iters": es.iterations, "e_s_ms": 1e3 * t_es,
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
        "cpu_baseline": cpu,
        "levels": [{k: lv[k] for k in ("level", "S", "p", "q", "rho_max", "t_eliminate_ms", "t_precondition_ms",
                                       "t_id_ms", "t_skel_update_ms", "t_repack_ms")} for lv in stats["levels"]],
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c5", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    args = ap.parse_args()
    world, rank, local, pg = dist_setup(args)
    try:
        if args.impl == "reference":
            run_reference(args, world, rank, pg)
        else:
            run_b200(args, world, rank, local, pg)
    finally:
        if pg is not None:
            pg.barrier()
            pg.destroy_process_group()


if __name__ == "__main__":
    main()
