#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab45_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab45_pytest.log
for r in 1 2; do
FT_NO_ODE1=1 timeout 300 python bench.py --config 1 --steps 5 --warmup 3 --no-cpu > gpurun_out/ab45_off_$r.json 2>gpurun_out/ab45_off.err
timeout 300 python bench.py --config 1 --steps 5 --warmup 3 --no-cpu > gpurun_out/ab45_on_$r.json 2>gpurun_out/ab45_on.err
done
