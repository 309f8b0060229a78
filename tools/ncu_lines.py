"""Top source lines by warp-stall samples from an ncu report: python tools/ncu_lines.py rep.ncu-rep [N]"""
import csv, subprocess, sys
rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname, lst, tot = "?", [], 0.0
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 5 or r[0] == "Line No":
        continue
    try:
        v = float(r[4])
    except ValueError:
        continue
    if r[2] != "-":          # SASS rows repeat the samples of their CUDA line
        continue
    tot += v
    lst.append((v, f"{fname}:{r[0]}", r[1].strip()[:100]))
lst.sort(reverse=True)
for v, loc, src in lst[:N]:
    print(f"{100 * v / max(tot, 1):5.1f}%  {loc:18s} {src}")
