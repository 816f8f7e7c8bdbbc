#!/bin/bash
# round evidence: full GPU tests, smoke, default bench (+e2e, cpu baseline), reference arm,
# ncu launch list of one solve, full captures of the main kernels (summarised on the box)
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/ev_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/ev_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ev_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/ev_bench_ref.json 2> gpurun_out/ev_bench_ref.err
python scratch/prof.py > gpurun_out/ev_prof.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/ev_launches.csv python scratch/prof.py > gpurun_out/ev_ncu_launch.log 2>&1
python scratch/launch_summary.py /tmp/ev_launches.csv > gpurun_out/ev_launch_summary.txt 2>&1
gzip -c /tmp/ev_launches.csv > gpurun_out/ev_launches.csv.gz
mkdir -p /tmp/ncu
for spec in "leaf_fused:100:leaffused" "mp_direct_kernel:300:mpdirect" "mp1g_kernel:40:mp1g9" "mp1g_kernel:190:mp1g11" "mp_kernel:0:mpcl2" "mp_kernel:1:mpcl4" "mp_kernel:10:mpsplit8" "mpB_kernel:0:mpB" "mp_fold_kernel:0:mpfold"; do
  IFS=: read k s name <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 -o /tmp/ncu/ev_$name python scratch/prof.py > gpurun_out/ev_$name.log 2>&1
  ncu -i /tmp/ncu/ev_$name.ncu-rep --page raw --csv > gpurun_out/ev_${name}_raw.csv 2>/dev/null
  ncu -i /tmp/ncu/ev_$name.ncu-rep --page source --csv --print-source sass > /tmp/ncu/ev_${name}_sass.csv 2>/dev/null
  gzip -c /tmp/ncu/ev_${name}_sass.csv > gpurun_out/ev_${name}_sass.csv.gz
done
cp /tmp/ncu/ev_leaffused.ncu-rep /tmp/ncu/ev_mp1g9.ncu-rep gpurun_out/ 2>/dev/null
du -sh gpurun_out
