#!/bin/bash
# round-2 cycle: all GPU tests, then the default bench (config 4) and config 5
cd $GRAFT_REPO_ROOT
P=${P:-r2d}
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/${P}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${P}_tests.log
timeout 900 python bench.py --config 5 --steps 2 --warmup 1 > gpurun_out/${P}_bench_c5.json 2> gpurun_out/${P}_bench_c5.err
timeout 600 python bench.py --config 2 --steps 20 > gpurun_out/${P}_bench_c2.json 2> gpurun_out/${P}_bench_c2.err
