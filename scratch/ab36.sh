#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scheme2.py -k "fused or multislab or wide or every_level" -q > gpurun_out/ab36_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab36_pytest.log
timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/ab36.json 2>gpurun_out/ab36.err
