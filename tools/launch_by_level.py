"""Per-level kernel totals from an ncu launch list of one factorization (levels split at k_repack / k_ingest)."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
seq = [(r[ki].split("(")[0].replace("void ", "").replace("phif::", ""), float(r[vi].replace(",", "")))
       for r in rows[hi + 1:] if len(r) > vi]
lev, per = -1, collections.defaultdict(collections.Counter)
for n, v in seq:
    if n in ("k_ingest", "k_repack"):
        lev += 1
    per[lev][n] += v
for l in sorted(per):
    tot = sum(per[l].values())
    top = ", ".join(f"{n} {v / 1e6:.1f}" for n, v in per[l].most_common(7))
    print(f"level {l}: {tot / 1e6:.1f} ms | {top}")
