#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --config 1 --steps 3000 --warmup 3 --e2e-steps 200 > gpurun_out/final3_cfg1.json 2>gpurun_out/final3_cfg1.err
timeout 900 python bench.py > gpurun_out/final3_bench.json 2>gpurun_out/final3_bench.err
