#!/bin/bash
# round-2 cycle: all GPU tests, default bench (config 4 + CPU baseline), configs 2, 3 and 5
cd $GRAFT_REPO_ROOT
P=${P:-r2f}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${P}_smi.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu -x --durations=25 > gpurun_out/${P}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${P}_tests.log
timeout 900 python bench.py > gpurun_out/${P}_bench_default.json 2> gpurun_out/${P}_bench_default.err
timeout 600 python bench.py --config 2 --steps 20 > gpurun_out/${P}_bench_c2.json 2> gpurun_out/${P}_bench_c2.err
timeout 600 python bench.py --config 3 --steps 10 > gpurun_out/${P}_bench_c3.json 2> gpurun_out/${P}_bench_c3.err
timeout 900 python bench.py --config 5 --steps 2 --warmup 1 > gpurun_out/${P}_bench_c5.json 2> gpurun_out/${P}_bench_c5.err
timeout 600 python bench.py --impl reference > gpurun_out/${P}_bench_ref.json 2> gpurun_out/${P}_bench_ref.err
nproc > gpurun_out/${P}_nproc.txt
