#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c2_pytest.log
timeout 600 python bench.py --no-cpu > gpurun_out/c2_bench.json 2> gpurun_out/c2_bench.err
