#!/bin/bash
cd $GRAFT_REPO_ROOT
for r in 1 2; do
  bash scratch/runvars.sh sync asy
  LEVELS_ARGS="--config 5" bash scratch/runvars.sh sync asy
done > gpurun_out/ab44.log 2>&1
cp scratch/var/asy/libfractime_b200.so paper_1710_11593_b200/libfractime_b200.so
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab44_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab44_pytest.log
