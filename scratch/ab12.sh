#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -k "fused_rhs or streamed" -x -q > gpurun_out/ab12_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab12_pytest.log
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu > gpurun_out/ab12_b.json 2>gpurun_out/ab12_b.err
