"""Per-launch list (in launch order) of one apply from an ncu CSV: python tools/apply_list.py launch_apply.csv"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
gi = h.index("Grid Size") if "Grid Size" in h else None
bi = h.index("Block Size") if "Block Size" in h else None
seq = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    d = seq.setdefault(r[ii], {})
    d[r[mi]] = float(r[vi].replace(",", ""))
    d["name"] = r[ki].split("(")[0]
    if gi is not None:
        d["grid"] = r[gi]
        d["block"] = r[bi]
for i, d in seq.items():
    t = d.get("gpu__time_duration.sum", 0)
    b = d.get("dram__bytes_read.sum", 0)
    print(f"{i:>5s} {d['name']:26s} grid {d.get('grid', ''):>16s} {t / 1e3:9.1f} us {b / 1e6:9.1f} MB {b / max(t, 1):7.0f} GB/s")
