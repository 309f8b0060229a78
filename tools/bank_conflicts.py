"""Per-kernel shared-memory bank-conflict share from an ncu CSV with the metrics
l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum, l1tex__data_pipe_lsu_wavefronts_mem_shared.sum, gpu__time_duration.sum."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.defaultdict(dict)
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
    per[r[ii]]["name"] = r[ki].split("(")[0].replace("void ", "").replace("phif::", "")
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for d in per.values():
    a = agg[d["name"]]
    a[0] += 1
    a[1] += d.get("gpu__time_duration.sum", 0)
    a[2] += d.get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 0)
    a[3] += d.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 0)
print(f"{'kernel':40s} {'n':>5s} {'ms':>9s} {'conflict wavefronts':>20s} {'share':>7s}")
for n, a in sorted(agg.items(), key=lambda x: -x[1][1])[:40]:
    print(f"{n[:40]:40s} {a[0]:5d} {a[1] / 1e6:9.2f} {a[2]:20.3g} {100 * a[2] / max(a[3], 1):6.1f}%")
