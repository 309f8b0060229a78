#!/bin/bash
# Round profiling on the GPU box: bench line, ncu launch list, ncu --set full of the top kernels.
# usage (via gpurun): bash tools/profile_round.sh r01
set -u
R=${1:-r01}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_c5_$R.json 2> gpurun_out/bench_c5_$R.err
echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_$R.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
# level-3 launch of the Gram-path CPQR (63 level-2 waves precede it) and of U = X^T X
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gid_cpqr --launch-skip 75 --launch-count 1 \
  -o gpurun_out/gidcpqr_l3_$R python tools/one_factor.py c5 1e-2 - 1 > gpurun_out/ncu_gid.log 2>&1
echo "gid full rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:k_big_nt<.int.1>" --launch-skip 2 --launch-count 1 \
  -o gpurun_out/bignt1_l3_$R python tools/one_factor.py c5 1e-2 - 1 > gpurun_out/ncu_bignt.log 2>&1
echo "big_nt full rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gid_gram --launch-skip 75 --launch-count 1 \
  -o gpurun_out/gidgram_l3_$R python tools/one_factor.py c5 1e-2 - 1 > gpurun_out/ncu_gram.log 2>&1
echo "gid gram full rc=$?"
