#!/bin/bash
# round evidence: plain bench, launch list of the same command, full captures of the main kernels
set -x
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ev_bench_small.json 2> gpurun_out/ev_bench_small.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ev_ncu_launch.log 2>&1
python scratch/prof.py > gpurun_out/ev_prof.log 2>&1 && {
ncu --set full --clock-control none --import-source on -k regex:mp1_kernel -s 40 -c 1 -o gpurun_out/ev_mp1 python scratch/prof.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:mp_direct -s 200 -c 1 -o gpurun_out/ev_mpdirect python scratch/prof.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:mp_kernel -s 0 -c 1 -o gpurun_out/ev_mpcluster python scratch/prof.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:mpB_kernel -s 0 -c 1 -o gpurun_out/ev_mpB python scratch/prof.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:leaf_kernel -s 100 -c 1 -o gpurun_out/ev_leaf python scratch/prof.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:leaf_correct -s 100 -c 1 -o gpurun_out/ev_leafcorrect python scratch/prof.py > /dev/null 2>&1
}
ls -la gpurun_out/ev_*
