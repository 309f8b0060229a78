import sys, time
sys.path.insert(0, ".")
from paper_1808_01364_b200.grid import baseline_problem
from paper_1808_01364_b200 import factorization as gf
from paper_1808_01364_b200.errors import NotSpdError
n = int(sys.argv[1]) if len(sys.argv) > 1 else None
for eps in (1e-4,):
    for seed in range(8):
        spec, A, _ = baseline_problem("c3", seed, n)
        t = time.time()
        try:
            F = gf.factorize(A, spec, eps, "phif")
            print("seed", seed, "eps", eps, "OK SL", F.SL, "%.2fs" % (time.time() - t), flush=True)
        except NotSpdError as e:
            print("seed", seed, "eps", eps, "NOTSPD", e.level, e.stage, e.group, e.pivot, "%.2fs" % (time.time() - t), flush=True)
