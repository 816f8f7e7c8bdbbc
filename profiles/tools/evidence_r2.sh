#!/bin/bash
# Round-2 evidence on one B200 (gpurun from the repo root): GPU tests, smoke,
# both bench arms, the ncu launch list of one config-4 solve, per-launch FP64 /
# DRAM of that solve, and one --set full capture per hot kernel.  Outputs under
# gpurun_out/ev2/ (summaries are copied into profiles/ncu_r02/ afterwards).
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/ev2; mkdir -p $O /tmp/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -s --junitxml=$O/pytest.xml -o junit_family=legacy > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err
timeout 1200 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
[ "$1" = "bench-only" ] && exit 0
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches.csv python profiles/tools/prof.py > $O/ncu_launch.log 2>&1
python profiles/tools/launch_summary.py /tmp/launches.csv > $O/launch_summary.md 2>&1
gzip -c /tmp/launches.csv > $O/launches_cfg4_solve.csv.gz
timeout 2400 ncu --metrics smsp__inst_executed_pipe_fp64.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"mp|leaf" --csv --log-file /tmp/fp64.csv python profiles/tools/prof.py > $O/fp64.log 2>&1
gzip -c /tmp/fp64.csv > $O/fp64_dram_per_launch_cfg4.csv.gz
cap() {  # name kernel-regex launch-skip [prof args]
  name=$1; k=$2; s=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$k" -s $s -c 1 -o /tmp/ncu/cap_$name -f python profiles/tools/prof.py "$@" > $O/cap_$name.log 2>&1
  ncu -i /tmp/ncu/cap_$name.ncu-rep --page raw --csv > $O/cap_${name}_raw.csv 2>/dev/null
  ncu -i /tmp/ncu/cap_$name.ncu-rep --page source --csv --print-source sass > /tmp/ncu/cap_${name}_sass.csv 2>/dev/null
  gzip -c /tmp/ncu/cap_${name}_sass.csv > $O/cap_${name}_sass.csv.gz
}
cap leaf_pair "leaf_pair" 100
FT_NO_PAIR=1 cap leaf_fused "leaf_fused" 100
cap split16 "mp_split_kernel<.int.16" 0
cap split8 "mp_split_kernel<.int.8," 0
cap cluster2 "mp_kernel<.int.2," 0
cap cluster4 "mp_kernel<.int.4," 0
cap mp1g9 "mp1g_kernel<.int.9>" 20
cap mp1g12 "mp1g_kernel<.int.12>" 4
cap direct64 "mp_direct_kernel" 300
cap ode_whole "ode_whole_kernel" 0 --config 1
cap leaf_cfg2 "leaf_kernel" 60 --config 2
cap leaf_cfg3 "leaf_chain" 60 --config 3 --time-steps 8192
cp /tmp/ncu/cap_leaf_pair.ncu-rep /tmp/ncu/cap_split16.ncu-rep $O/ 2>/dev/null
du -sh $O
