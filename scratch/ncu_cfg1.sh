#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_cfg1.csv python bench.py --config 1 --steps 5 --warmup 3 --no-cpu --e2e-steps 2 > gpurun_out/ncu_cfg1.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:ode_whole -c 1 -o gpurun_out/ode_whole_cfg1 python bench.py --config 1 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_cfg1_full.log 2>&1
echo done
