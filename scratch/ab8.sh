#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -k "multislab or full_width or every_level" -x -q > gpurun_out/ab8_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab8_pytest.log
timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/ab8_b.json 2>gpurun_out/ab8_b.err
FT_LEAF_DBG=4 python scratch/leafclk.py > gpurun_out/ab8_clk.log 2>&1
