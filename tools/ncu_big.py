"""Per-kernel totals (time, DMMA pipe % time-weighted) from an ncu csv with gpu__time_duration.sum +
sm__inst_executed_pipe_tensor_subpipe_dmma...; optional: list the largest launches."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ii, ki, mi, vi = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
L = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    d = L.setdefault(r[ii], {"name": r[ki].split("(")[0].replace("void ", "")})
    d[r[mi]] = float(r[vi].replace(",", ""))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for d in L.values():
    t = d.get("gpu__time_duration.sum", 0.0)
    p = d.get("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", 0.0)
    a = agg[d["name"]]
    a[0] += 1; a[1] += t; a[2] += t * p
for n, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{n:28s} {a[0]:5d} launches {a[1]/1e6:8.2f} ms  dmma {a[2]/max(a[1],1):5.1f}%")
if len(sys.argv) > 2:
    big = sorted(L.values(), key=lambda d: -d.get("gpu__time_duration.sum", 0))[: int(sys.argv[2])]
    for d in big:
        print(d["name"], "%.3f ms" % (d["gpu__time_duration.sum"] / 1e6), "grid", int(d.get("launch__grid_size", 0)),
              "dmma %.1f" % d.get("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", 0))
