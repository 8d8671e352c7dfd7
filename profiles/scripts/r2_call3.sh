#!/bin/bash
cd $GRAFT_REPO_ROOT
P=r2h
( cd profiles/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o upd_bench upd_bench.cu && timeout 120 ./upd_bench ) > gpurun_out/${P}_upd_bench.txt 2>&1
timeout 900 python profiles/eps_probe.py --config 2 > gpurun_out/${P}_eps_c2.txt 2>&1
timeout 900 python profiles/eps_probe.py --config 4 > gpurun_out/${P}_eps_c4.txt 2>&1
