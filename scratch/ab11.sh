#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -k "fused_rhs or multislab" -x -q > gpurun_out/ab11_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab11_pytest.log
timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/ab11_b.json 2>gpurun_out/ab11_b.err
