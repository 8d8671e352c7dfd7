#!/bin/bash
# round-2 check: full-size shell test, default bench (config 4 with its CPU baseline), configs 3 and 5
cd $GRAFT_REPO_ROOT
P=${P:-r2c}
timeout 900 python -m pytest tests/test_gpu_shell.py -q > gpurun_out/${P}_shell.log 2>&1
echo "rc=$?" >> gpurun_out/${P}_shell.log
timeout 900 python bench.py > gpurun_out/${P}_bench_default.json 2> gpurun_out/${P}_bench_default.err
timeout 600 python bench.py --config 3 --steps 10 > gpurun_out/${P}_bench_c3.json 2> gpurun_out/${P}_bench_c3.err
timeout 900 python bench.py --config 5 --steps 2 --warmup 1 > gpurun_out/${P}_bench_c5.json 2> gpurun_out/${P}_bench_c5.err
lscpu > gpurun_out/${P}_lscpu.txt; free -g >> gpurun_out/${P}_lscpu.txt
