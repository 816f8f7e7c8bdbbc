#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/ab33_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab33_pytest.log
