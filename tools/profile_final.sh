#!/bin/bash
# End-of-round profiling on the GPU box (bench lines, launch lists, ncu --set full of the top kernels).
# usage (via gpurun): bash tools/profile_final.sh r02
set -u
R=${1:-r02}
O=gpurun_out/final
mkdir -p $O
timeout 900 python bench.py > $O/bench_c5_$R.json 2> $O/bench_c5_$R.err; echo "bench c5 rc=$?"
timeout 900 python bench.py --workload c3p --no-cpu > $O/bench_c3p_$R.json 2> $O/bench_c3p_$R.err; echo "bench c3p rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref_$R.json 2> $O/bench_ref_$R.err; echo "bench ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5_$R.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu > $O/ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --profile-from-start off --csv \
  --log-file $O/launch_apply_$R.csv python tools/apply_probe.py 32 2 p > $O/ncu_apply.log 2>&1; echo "apply list rc=$?"
M=l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,gpu__time_duration.sum
timeout 900 ncu --metrics $M --clock-control none --csv --log-file $O/bank_c5_$R.csv python tools/one_factor.py c5 1e-2 - 1 > $O/bank.log 2>&1; echo "bank rc=$?"
# level-3 launches: wide trailing update, U = X^T X, TRSM; deep replay GEMM of the apply
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:k_big_nt<.int.0>" --launch-skip 110 --launch-count 1 \
  -o $O/bignt0_l3_$R python tools/one_factor.py c5 1e-2 - 1 > $O/ncu_bignt0.log 2>&1; echo "big_nt0 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_big_trsm --launch-skip 90 --launch-count 1 \
  -o $O/bigtrsm_l3_$R python tools/one_factor.py c5 1e-2 - 1 > $O/ncu_trsm.log 2>&1; echo "trsm rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_rgemm_deep --launch-skip 4 --launch-count 1 \
  -o $O/rgemm_deep_$R python tools/apply_probe.py 32 2 p > $O/ncu_rgemm.log 2>&1; echo "rgemm rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_apply_cell_mma --launch-count 1 \
  -o $O/apply_cell_mma_$R python tools/apply_probe.py 32 2 p > $O/ncu_cellmma.log 2>&1; echo "cell mma rc=$?"
timeout 1200 python -m pytest tests -x -q -m gpu > $O/gputest_$R.log 2>&1; echo "pytest rc=$?"; tail -2 $O/gputest_$R.log
