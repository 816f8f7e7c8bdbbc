#!/bin/bash
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/fin_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/fin_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/fin_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/fin_bench_ref.json 2> gpurun_out/fin_bench_ref.err
timeout 300 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu > gpurun_out/fin_cfg5.json 2> gpurun_out/fin_cfg5.err
