#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scheme2.py -x -q > gpurun_out/ab14_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab14_pytest.log
timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-fused > gpurun_out/ab14_tab.json 2>gpurun_out/ab14_tab.err
