#!/bin/bash
# round check: gpu tests, smoke, full bench, launch list of a short bench
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/rc_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/rc_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rc_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/rc_bench.json 2> gpurun_out/rc_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/rc_bench_ref.json 2> gpurun_out/rc_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rc_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/rc_ncu_launch.log 2>&1
ls -la gpurun_out
