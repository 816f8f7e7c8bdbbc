#!/bin/bash
cd $GRAFT_REPO_ROOT
run() { name=$1; shift; env "$@" timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/ab2_$name.json 2>gpurun_out/ab2_$name.err; }
run def FT_X=1
run k8cl FT_SPLIT_MIN_K=16
run allcl FT_CLUSTER_K=1
FT_SPLIT_MIN_K=16 timeout 600 python -m pytest tests/test_gpu_parity.py -k "every_level" -x -q > gpurun_out/ab2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab2_pytest.log
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scheme2.py -k "every_level or long_run" -x -q >> gpurun_out/ab2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab2_pytest.log
