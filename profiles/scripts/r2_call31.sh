#!/bin/bash
# final-state lines for configs 1 and 5
cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --config 1 --steps 20 > gpurun_out/r2x8_bench_c1.json 2> gpurun_out/r2x8_bench_c1.err
( time timeout 1500 python bench.py --config 5 --steps 1 --warmup 1 > gpurun_out/r2x8_bench_c5.json 2> gpurun_out/r2x8_bench_c5.err ) 2> gpurun_out/r2x8_time.txt
