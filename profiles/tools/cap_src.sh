#!/bin/bash
# One ncu --set full capture of one kernel launch with the per-instruction SASS page.
# usage: cap_src.sh <name> <kernel-regex> <launch-skip> [lab.py args]   (outputs under gpurun_out/cap/)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/cap; mkdir -p $O /tmp/ncu
name=$1; k=$2; s=$3; shift 3
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$k" -s $s -c 1 -o /tmp/ncu/cap_$name -f python profiles/tools/prof.py "$@" > $O/cap_$name.log 2>&1
ncu -i /tmp/ncu/cap_$name.ncu-rep --page raw --csv > $O/cap_${name}_raw.csv 2>/dev/null
ncu -i /tmp/ncu/cap_$name.ncu-rep --page source --csv --print-source sass > /tmp/ncu/cap_${name}_sass.csv 2>/dev/null
gzip -c /tmp/ncu/cap_${name}_sass.csv > $O/cap_${name}_sass.csv.gz
ls -la $O
