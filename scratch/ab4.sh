#!/bin/bash
cd $GRAFT_REPO_ROOT
run() { name=$1; shift; env "$@" timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/ab4_$name.json 2>gpurun_out/ab4_$name.err; }
run pdl0 FT_X=1
run pdl1 FT_PDL=1
run pdl2 FT_PDL=2
FT_PDL=2 timeout 600 python -m pytest tests/test_gpu_parity.py -k "every_level or multislab or full_width" -x -q > gpurun_out/ab4_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab4_pytest.log
