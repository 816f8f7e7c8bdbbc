#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scheme2.py tests/test_parallel.py -x -q > gpurun_out/ab39_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab39_pytest.log
timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-fused > gpurun_out/ab39.json 2>gpurun_out/ab39.err
timeout 300 python bench.py --config 3 --steps 5 --warmup 3 --no-e2e --no-cpu --no-fused > gpurun_out/ab39_c3.json 2>gpurun_out/ab39_c3.err
FT_LEAF_DBG=4 python scratch/leafclk.py > gpurun_out/ab39_clk.log 2>&1
