#!/bin/bash
# Build libphif_b200.so for sm_100a (in-tree, travels with the gpurun snapshot).
set -euo pipefail
cd "$(dirname "$0")"
OUT=../libphif_b200.so
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
FLAGS="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC,-O3,-g,-fopenmp --expt-relaxed-constexpr"
mkdir -p build
# the translation units are independent: compile them concurrently
pids=()
$NVCC $FLAGS -c planner.cpp -o build/planner.o & pids+=($!)
$NVCC $FLAGS -c kernels.cu -o build/kernels.o ${PTXAS_V:+-Xptxas -v} & pids+=($!)
$NVCC $FLAGS -c engine.cu -o build/engine.o & pids+=($!)
$NVCC $FLAGS -c gpu_plan.cu -o build/gpu_plan.o & pids+=($!)
$NVCC $FLAGS -c problem.cu -o build/problem.o & pids+=($!)
$NVCC $FLAGS -c capi.cu -o build/capi.o & pids+=($!)
for p in "${pids[@]}"; do wait "$p"; done
$NVCC -shared -gencode arch=compute_100a,code=sm_100a -o $OUT build/planner.o build/kernels.o build/engine.o build/gpu_plan.o build/problem.o build/capi.o -lcudart -lgomp -Xlinker -export-dynamic
echo "built $(realpath $OUT)"
