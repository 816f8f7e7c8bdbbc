#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_parallel.py -x -q > gpurun_out/ab38_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab38_pytest.log
timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-fused > gpurun_out/ab38.json 2>gpurun_out/ab38.err
FT_NO_FUSE0=1 timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-fused > gpurun_out/ab38_nf.json 2>gpurun_out/ab38_nf.err
FT_LEAF_DBG=4 python scratch/leafclk.py > gpurun_out/ab38_clk.log 2>&1
