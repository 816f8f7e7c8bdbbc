#!/bin/bash
cd $GRAFT_REPO_ROOT
cp paper_1710_11593_b200/libfractime_b200.so /tmp/lib_orig.so
for v in base u1 u4; do
  if [ $v != base ]; then cp scratch/var/$v/libfractime_b200.so paper_1710_11593_b200/libfractime_b200.so; fi
  timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-fused > gpurun_out/ab16_$v.json 2>gpurun_out/ab16_$v.err
  cp /tmp/lib_orig.so paper_1710_11593_b200/libfractime_b200.so
done
