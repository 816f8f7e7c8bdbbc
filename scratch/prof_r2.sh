#!/bin/bash
cd $GRAFT_REPO_ROOT
python scratch/prof.py > gpurun_out/p2_prof.log 2>&1 || exit 1
for spec in "mp1g_kernel:40:mp1g" "leaf_kernel:100:leaf" "leaf_correct:100:leafcorrect" "mp_kernel:1:mpsplit" "mp1_kernel:0:mp1_13" "mp_direct:300:mpdirect"; do
  IFS=: read k s name <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 -o gpurun_out/p2_$name python scratch/prof.py > gpurun_out/p2_$name.log 2>&1
done
ls -la gpurun_out/
