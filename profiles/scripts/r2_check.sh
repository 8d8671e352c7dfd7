#!/bin/bash
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2b_smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -k "not full_size" > gpurun_out/r2b_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2b_tests.log
for c in 2 4; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_bench_c$c.json 2> gpurun_out/r2b_bench_c$c.err
done
