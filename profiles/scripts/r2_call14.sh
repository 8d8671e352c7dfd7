#!/bin/bash
cd $GRAFT_REPO_ROOT
P=r2s
timeout 900 python profiles/c5_newton_diag.py 20 > gpurun_out/${P}_c5newton.txt 2>&1
timeout 1500 python bench.py --config 5 --steps 1 --warmup 1 > gpurun_out/${P}_c5.json 2> gpurun_out/${P}_c5.err
timeout 900 python -m pytest -q tests/test_gpu_shell.py > gpurun_out/${P}_shell.log 2>&1
