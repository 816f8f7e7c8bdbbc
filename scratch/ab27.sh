#!/bin/bash
cd $GRAFT_REPO_ROOT
FT_SMALL_NPT2=1 timeout 600 python -m pytest tests/test_gpu_parity.py -k "cfg2 or golden or paper" -x -q > gpurun_out/ab27_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab27_pytest.log
for v in base npt2; do
  if [ $v = npt2 ]; then export FT_SMALL_NPT2=1; fi
  timeout 300 python bench.py --config 2 --steps 5 --warmup 3 --no-e2e --no-cpu --no-fused > gpurun_out/ab27_$v.json 2>gpurun_out/ab27_$v.err
done
