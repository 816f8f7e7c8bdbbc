#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab10_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab10_pytest.log
run() { name=$1; shift; env "$@" timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/ab10_$name.json 2>gpurun_out/ab10_$name.err; }
run pf FT_X=1
run nopf FT_LEAF_DBG=16
