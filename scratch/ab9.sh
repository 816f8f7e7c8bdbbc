#!/bin/bash
cd $GRAFT_REPO_ROOT
FT_FUSED_LEAF=1 timeout 600 python -m pytest tests/test_gpu_parity.py -k "multislab or full_width or streamed" -x -q > gpurun_out/ab9_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab9_pytest.log
run() { name=$1; shift; env "$@" timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/ab9_$name.json 2>gpurun_out/ab9_$name.err; }
run fused FT_FUSED_LEAF=1
run plain FT_X=1
