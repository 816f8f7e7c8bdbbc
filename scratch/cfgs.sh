#!/bin/bash
cd $GRAFT_REPO_ROOT
for c in 1 2 3 5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
done
