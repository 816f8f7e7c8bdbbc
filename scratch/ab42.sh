#!/bin/bash
cd $GRAFT_REPO_ROOT
for r in 1 2; do
  bash scratch/runvars.sh d256 d128 d512
  LEVELS_ARGS="--config 5" bash scratch/runvars.sh d256 d128 d512
done > gpurun_out/ab42.log 2>&1
