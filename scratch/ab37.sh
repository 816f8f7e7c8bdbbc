#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scheme2.py -x -q > gpurun_out/ab37_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab37_pytest.log
cp paper_1710_11593_b200/libfractime_b200.so /tmp/lib_orig.so
for v in async sync async2; do
  if [ $v = sync ]; then cp scratch/var/sync/libfractime_b200.so paper_1710_11593_b200/libfractime_b200.so; fi
  timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-fused > gpurun_out/ab37_$v.json 2>gpurun_out/ab37_$v.err
  cp /tmp/lib_orig.so paper_1710_11593_b200/libfractime_b200.so
done
FT_LEAF_DBG=4 python scratch/leafclk.py > gpurun_out/ab37_clk.log 2>&1
