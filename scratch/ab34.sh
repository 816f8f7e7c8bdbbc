#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -k "harness" -q > gpurun_out/ab34_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab34_pytest.log
python -m paper_1710_11593_b200.harness --example 2 --gamma 0.1 0.9 --levels 3..8 --fixed-tau-exp 10 --format markdown > gpurun_out/ab34_ex2.md 2>&1
