#!/bin/bash
cd $GRAFT_REPO_ROOT
P=${P:-r2e}
timeout 900 python profiles/c5_profile.py --instances 8 > gpurun_out/${P}_c5prof8.txt 2>&1
timeout 900 python profiles/c5_profile.py --instances 64 > gpurun_out/${P}_c5prof64.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_shell.py tests/test_gpu_minimize_batched.py tests/test_gpu_large.py tests/test_gpu_sgn.py -q -s > gpurun_out/${P}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${P}_tests.log
