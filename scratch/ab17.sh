#!/bin/bash
cd $GRAFT_REPO_ROOT
FT_SLAB_MIN=513 timeout 900 python -m pytest tests/test_gpu_parity.py -k "cfg3 or cfg2 or every_level" -x -q > gpurun_out/ab17_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab17_pytest.log
for c in 3 2; do
for sm in 2049 513 257; do
  FT_SLAB_MIN=$sm timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu --no-fused > gpurun_out/ab17_c${c}_$sm.json 2>gpurun_out/ab17_c${c}_$sm.err
done; done
