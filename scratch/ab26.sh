#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_parallel.py -x -q > gpurun_out/ab26_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab26_pytest.log
run() { name=$1; shift; env "$@" timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-fused > gpurun_out/ab26_$name.json 2>gpurun_out/ab26_$name.err; }
run fuse0 FT_X=1
run nofuse0 FT_NO_FUSE0=1
run fuse0b FT_X=1
