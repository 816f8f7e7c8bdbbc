#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab7_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab7_pytest.log
run() { name=$1; shift; env "$@" timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/ab7_$name.json 2>gpurun_out/ab7_$name.err; }
run kc FT_X=1
run nokc FT_NO_KC=1
FT_LEAF_DBG=4 python scratch/leafclk.py > gpurun_out/ab7_clk.log 2>&1
