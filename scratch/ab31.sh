#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-fused > gpurun_out/ab31.json 2>gpurun_out/ab31.err
