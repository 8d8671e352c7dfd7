#!/bin/bash
# config 5 bench line (one batched 20-iteration run of 64 instances per step)
cd $GRAFT_REPO_ROOT
P=${P:-r2c5}
( time timeout 2700 python bench.py --config 5 --steps 1 --warmup 1 > gpurun_out/${P}_bench_c5.json 2> gpurun_out/${P}_bench_c5.err ) 2> gpurun_out/${P}_time.txt
