#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/ab20_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab20_pytest.log
timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-fused > gpurun_out/ab20_c4.json 2>gpurun_out/ab20_c4.err
