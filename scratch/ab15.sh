#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scheme2.py tests/test_gpu_toeplitz.py -x -q > gpurun_out/ab15_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab15_pytest.log
run() { name=$1; shift; env "$@" timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-fused > gpurun_out/ab15_$name.json 2>gpurun_out/ab15_$name.err; }
run persist FT_X=1
run plain FT_MP1_NOPERSIST=1
