#!/bin/bash
cd $GRAFT_REPO_ROOT
P=r2p2
timeout 600 python profiles/small_shell_diag.py > gpurun_out/${P}_small_shell.txt 2>&1
timeout 1200 python bench.py --config 5 --steps 1 --warmup 1 > gpurun_out/${P}_c5.json 2> gpurun_out/${P}_c5.err
