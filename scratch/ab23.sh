#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -k "edge_shapes" -q > gpurun_out/ab23_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab23_pytest.log
