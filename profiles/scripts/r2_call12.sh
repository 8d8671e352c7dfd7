#!/bin/bash
cd $GRAFT_REPO_ROOT
P=r2q
timeout 900 python profiles/c5_newton_diag.py 10 > gpurun_out/${P}_c5newton.txt 2>&1
timeout 900 python -m pytest -q tests/test_gpu_shell.py > gpurun_out/${P}_shell.log 2>&1
timeout 600 python profiles/c4_parity_diag.py > gpurun_out/${P}_c4diag.txt 2>&1
