set -x
timeout 900 python -m pytest tests/test_gpu_planner.py -x -q > gpurun_out/r2b_planner.txt 2>&1
python tools/one_factor.py c5 1e-2 - 4 -v > gpurun_out/r2b_onefactor.txt 2>&1
PHIF_DEBUG=1 python tools/one_factor.py c5 1e-2 - 2 > gpurun_out/r2b_debug.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_fullsize_oracle.py > gpurun_out/r2b_pytest.txt 2>&1
tail -3 gpurun_out/r2b_pytest.txt gpurun_out/r2b_planner.txt
