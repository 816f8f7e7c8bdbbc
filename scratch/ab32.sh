#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_scheme2.py -q > gpurun_out/ab32_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab32_pytest.log
