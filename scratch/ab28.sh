#!/bin/bash
cd $GRAFT_REPO_ROOT
cp paper_1710_11593_b200/libfractime_b200.so /tmp/lib_orig.so
for v in base ch16 ch4; do
  if [ $v != base ]; then cp scratch/var/$v/libfractime_b200.so paper_1710_11593_b200/libfractime_b200.so; fi
  timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-fused > gpurun_out/ab28_$v.json 2>gpurun_out/ab28_$v.err
  timeout 300 python -m pytest tests/test_gpu_parity.py -k "every_level" -x -q > gpurun_out/ab28_$v.pytest 2>&1
  cp /tmp/lib_orig.so paper_1710_11593_b200/libfractime_b200.so
done
