#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_parallel.py -x -q > gpurun_out/ab13_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab13_pytest.log
run() { name=$1; shift; env "$@" timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-fused > gpurun_out/ab13_$name.json 2>gpurun_out/ab13_$name.err; }
run lr FT_X=1
run full FT_FULL_PHASE3=1
FT_LEAF_DBG=4 FT_NO_FUSED_LEAF=1 python scratch/leafclk.py > gpurun_out/ab13_clk.log 2>&1
