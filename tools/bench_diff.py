"""Side-by-side of two bench lines: step time, per-(level, stage) times."""
import json, sys
ds = [json.loads(open(f).read().strip().splitlines()[-1]) for f in sys.argv[1:]]
for f, d in zip(sys.argv[1:], ds):
    print(f, "ms/step %.1f  plan %.1f  solve %.2f ms/rhs  frac %.3f (%s %.2f ms)" % (
        d["ms_per_step"], d["t_plan_ms"], d["solve_ms_per_rhs"], d["roofline"]["frac"], d["roofline"]["kernel"],
        d["roofline"]["time_ms"]))
keys = [(r["level"], r["stage"]) for r in ds[0]["roofline_levels"]]
tab = [{(r["level"], r["stage"]): r for r in d["roofline_levels"]} for d in ds]
for k in keys:
    print("%d %-13s" % k, "  ".join("%7.2f ms %5.1f%%" % (t[k]["t_ms"], 100 * t[k]["frac_fp64"]) if k in t else "-" for t in tab))
print("sum           ", "  ".join("%7.2f ms" % sum(r["t_ms"] for r in t.values()) for t in tab))
