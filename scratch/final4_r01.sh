#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final4_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/final4_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final4_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final4_smoke.log
timeout 300 python bench.py --config 1 --steps 3000 --warmup 3 --e2e-steps 200 > gpurun_out/final4_cfg1.json 2>gpurun_out/final4_cfg1.err
