#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-fused > gpurun_out/ab35.json 2>gpurun_out/ab35.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ab35_smoke.log 2>&1
