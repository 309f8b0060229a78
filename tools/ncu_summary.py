"""Summarize an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel count, total, share."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0]
    unit_scale = 1.0
    v = float(r[vi].replace(",", ""))
    tot[name] += v; cnt[name] += 1
unit = rows[hdr_i + 1][hdr.index("Metric Unit")] if "Metric Unit" in hdr else "?"
T = sum(tot.values())
print(f"total {T:.4g} {unit} over {sum(cnt.values())} launches")
print(f"{'kernel':40s} {'launches':>8s} {'total':>12s} {'share':>7s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k:40s} {cnt[k]:8d} {v:12.4g} {100*v/T:6.1f}%")
