#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p /tmp/ncu
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mp_direct_kernel -s 40 -c 1 -o /tmp/ncu/dir64 python scratch/prof.py > gpurun_out/dir64.log 2>&1
ncu -i /tmp/ncu/dir64.ncu-rep --page raw --csv > gpurun_out/dir64_raw.csv 2>/dev/null
ncu -i /tmp/ncu/dir64.ncu-rep --page source --csv --print-source sass > gpurun_out/dir64_sass.csv 2>/dev/null
ncu -i /tmp/ncu/dir64.ncu-rep --page details --csv > gpurun_out/dir64_details.csv 2>/dev/null
gzip -f gpurun_out/dir64_sass.csv
