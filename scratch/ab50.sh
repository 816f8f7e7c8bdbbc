#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab50_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab50_pytest.log
cp paper_1710_11593_b200/libfractime_b200.so /tmp/lib_orig.so
for r in 1 2; do for v in o9 o10; do
  cp scratch/var/$v/libfractime_b200.so paper_1710_11593_b200/libfractime_b200.so
  timeout 300 python bench.py --config 1 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab50_${v}_$r.json 2>/dev/null
done; done
cp /tmp/lib_orig.so paper_1710_11593_b200/libfractime_b200.so
