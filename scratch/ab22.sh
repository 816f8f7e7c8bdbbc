#!/bin/bash
cd $GRAFT_REPO_ROOT
for v in "1 2048" "2 2048" "4 2048" "2 4096"; do
  set -- $v
  echo "streams=$1 chunk=$2" >> gpurun_out/ab22.log
  FT_D2H_STREAMS=$1 FT_STREAM_CHUNK=$2 timeout 300 python scratch/e2e_ab.py >> gpurun_out/ab22.log 2>&1
done
FT_D2H_STREAMS=2 timeout 600 python -m pytest tests/test_gpu_parity.py -k "streamed" -x -q >> gpurun_out/ab22.log 2>&1
