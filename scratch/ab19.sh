#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scheme2.py -k "every_level or long_run or multislab or fused" -x -q > gpurun_out/ab19_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab19_pytest.log
run() { name=$1; shift; env "$@" timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-fused > gpurun_out/ab19_$name.json 2>gpurun_out/ab19_$name.err; }
run serial FT_SPLIT_SERIAL=1
run pipe128 FT_X=1
run pipe64 FT_MP_BATCH_MB=64
run pipe32 FT_MP_BATCH_MB=32
