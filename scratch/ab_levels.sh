#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -k "every_level or multislab" tests/test_gpu_scheme2.py -k "every_level or long_run or multislab" -x -q > gpurun_out/ab_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab_pytest.log
FT_SINGLE_MAX=4096 FT_SPLIT_MIN_K=2 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scheme2.py -k "every_level or long_run" -x -q >> gpurun_out/ab_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab_pytest.log
FT_SINGLE_MAX=4096 timeout 600 python -m pytest tests/test_gpu_parity.py -k "every_level" -x -q >> gpurun_out/ab_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab_pytest.log
run() { name=$1; shift; env "$@" timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/ab_$name.json 2>gpurun_out/ab_$name.err; }
run base FT_NO_PREFOLD=1
run prefold FT_X=1
run pf64 FT_MP_BATCH_MB=64
run pf128 FT_MP_BATCH_MB=128
run pfk4 FT_SPLIT_MIN_K=4
run pfk4b64 FT_SPLIT_MIN_K=4 FT_MP_BATCH_MB=64
run s4096c FT_SINGLE_MAX=4096
run s4096s FT_SINGLE_MAX=4096 FT_SPLIT_MIN_K=2
run s4096s64 FT_SINGLE_MAX=4096 FT_SPLIT_MIN_K=2 FT_MP_BATCH_MB=64
