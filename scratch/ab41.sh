#!/bin/bash
# L2 prefetch of the next leaf's tile: on vs off (FT_NO_LEAF_PF)
cd $GRAFT_REPO_ROOT
B="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-fused"
for r in 1 2; do
  for c in 4 3 5; do
    FT_NO_LEAF_PF=1 timeout 300 $B --config $c > gpurun_out/ab41_off_c${c}_$r.json 2>/dev/null
    timeout 300 $B --config $c > gpurun_out/ab41_on_c${c}_$r.json 2>/dev/null
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scheme2.py -x -q > gpurun_out/ab41_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab41_pytest.log
