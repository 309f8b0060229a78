"""Summarise an ncu launch list (time + dram read) of one apply: python tools/apply_launches.py launch_apply.csv"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
seqd = collections.defaultdict(dict)
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    seqd[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
    seqd[r[ii]]["name"] = r[ki].split("(")[0]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for d in seqd.values():
    a = agg[d["name"]]
    a[0] += 1
    a[1] += d.get("gpu__time_duration.sum", 0)
    a[2] += d.get("dram__bytes_read.sum", 0)
T = sum(a[1] for a in agg.values())
B = sum(a[2] for a in agg.values())
print(f"apply kernels total {T / 1e6:.2f} ms, dram read {B / 1e9:.2f} GB ({B / T:.0f} GB/s)")
for n, a in sorted(agg.items(), key=lambda x: -x[1][1])[:10]:
    print(f"{n:28s} {a[0]:4d} {a[1] / 1e6:8.2f} ms {a[2] / 1e9:7.2f} GB {a[2] / max(a[1], 1):6.0f} GB/s")
