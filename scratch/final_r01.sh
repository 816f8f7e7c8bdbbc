#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final_smoke.log
for c in 1 2 3 5; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/final_cfg$c.json 2>gpurun_out/final_cfg$c.err; done
timeout 900 python bench.py > gpurun_out/final_bench.json 2>gpurun_out/final_bench.err
