#!/bin/bash
# batched leaf: in-leaf weights via constant cache (wc) vs registers (wreg)
cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in wreg wc; do
  cp scratch/var/$v/libfractime_b200.so paper_1710_11593_b200/libfractime_b200.so
  timeout 300 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu --no-fused > gpurun_out/ab40_${v}_$r.json 2>gpurun_out/ab40_${v}_$r.err
done; done
cp scratch/var/wc/libfractime_b200.so paper_1710_11593_b200/libfractime_b200.so
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab40_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab40_pytest.log
