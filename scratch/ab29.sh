#!/bin/bash
cd $GRAFT_REPO_ROOT
for v in fuse0 nofuse0; do
  if [ $v = nofuse0 ]; then export FT_NO_FUSE0=1; fi
  timeout 300 python bench.py --config 3 --steps 5 --warmup 3 --no-e2e --no-cpu --no-fused > gpurun_out/ab29_$v.json 2>gpurun_out/ab29_$v.err
done
