#!/bin/bash
cd $GRAFT_REPO_ROOT
P=r2j
timeout 900 python profiles/c4_parity_diag.py > gpurun_out/${P}_c4diag.txt 2>&1
timeout 600 python profiles/fdag_trace.py --config 4 --summary --out /tmp/t4.npz > gpurun_out/${P}_trace_c4.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/${P}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${P}_tests.log
