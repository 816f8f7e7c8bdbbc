#!/bin/bash
# FP64 work of one config-4 solve: per-launch FP64 pipe instructions and DRAM bytes (ncu, all solve kernels)
cd $GRAFT_REPO_ROOT
timeout 2400 ncu --metrics smsp__inst_executed_pipe_fp64.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"mp|leaf" --csv --log-file /tmp/fp64.csv python scratch/prof.py > gpurun_out/fp64_ncu.log 2>&1
gzip -c /tmp/fp64.csv > gpurun_out/fp64_solve.csv.gz
