"""bench_cli: argument handling, exit codes, CSV schema, scaling fits (CPU), and
one bench sweep on the GPU (HIF vs PHIF rows, NotSpd reported as data)."""
import csv
import json
import os

import numpy as np
import pytest

from conftest import gpu_available
from paper_1808_01364_b200 import cli


def test_csv_header_is_spec():
    assert ",".join(cli.CSV_HEADER) == "method,eps,dim,n,N,seed,SL,e_a,e_s,n_i,t_factor_s,t_apply_s,mem_bytes,status"


def test_unknown_flag_exits_64():
    with pytest.raises(SystemExit) as e:
        cli.main(["factor", "--bogus"])
    assert e.value.code == 64


def test_scaling_slopes(tmp_path):
    rows = []
    for N, t in ((1000, 1.0), (4000, 4.0), (16000, 16.0)):
        rows.append({"method": "phif", "N": N, "t_factor_s": t, "t_apply_s": t / 10, "mem_bytes": 8 * N,
                     "status": "ok"})
    res = cli.emit_scaling(rows)
    assert abs(res["slopes"]["phif"]["factor_time"] - 1.0) < 0.05
    assert len(res["rows"]) == 3
    with pytest.raises(ValueError):
        cli.emit_scaling(rows[:1])
    p = tmp_path / "r.csv"
    with open(p, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=cli.CSV_HEADER)
        w.writeheader()
        for r in rows:
            w.writerow({k: r.get(k, "") for k in cli.CSV_HEADER})
    assert cli.main(["scaling", str(p), "--out", str(tmp_path / "s.json")]) == 0
    assert json.load(open(tmp_path / "s.json"))["slopes"]["phif"]["memory"] == pytest.approx(1.0, abs=1e-9)


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")
def test_bench_rows_hif_vs_phif(tmp_path):
    out = tmp_path / "b.csv"
    rc = cli.main(["bench", "--dim", "2", "--n", "64", "--m", "8", "--eps-list", "1e-6", "--methods", "hif,phif,exact",
                   "--seeds", "2", "--out", str(out)])
    assert rc == 0
    rows = list(csv.DictReader(open(out)))
    assert list(rows[0].keys()) == cli.CSV_HEADER and len(rows) == 6
    ex = [r for r in rows if r["method"] == "exact"]
    assert all(float(r["e_s"]) <= 1e-9 and int(r["n_i"]) <= 2 for r in ex)
    ph = [r for r in rows if r["method"] == "phif"]
    hf = [r for r in rows if r["method"] == "hif"]
    assert np.median([float(r["e_s"]) for r in ph]) < np.median([float(r["e_s"]) for r in hf])
    # a NotSpd factorization is data: status not-spd, exit code 2 for `factor`
    assert cli.main(["factor", "--config", "c3", "--n", "256", "--seed", "1", "--eps", "1e-2"]) == 2
