#!/bin/bash
cd $GRAFT_REPO_ROOT
P=r2r
timeout 900 python profiles/c5_newton_diag.py 5 > gpurun_out/${P}_c5newton.txt 2>&1
