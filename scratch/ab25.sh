#!/bin/bash
cd $GRAFT_REPO_ROOT
FT_RADIX8=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scheme2.py -x -q > gpurun_out/ab25_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab25_pytest.log
run() { name=$1; shift; env "$@" timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-fused > gpurun_out/ab25_$name.json 2>gpurun_out/ab25_$name.err; }
run r8 FT_RADIX8=1
run r16 FT_X=1
