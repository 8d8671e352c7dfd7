#!/bin/bash
# quick cycle: factor/solve tests, config 4/3/2 bench lines without the CPU leg, config-4 task trace
cd $GRAFT_REPO_ROOT
P=${P:-r2r}
timeout 900 python -m pytest tests/test_gpu_linear.py tests/test_gpu_sgn.py tests/test_gpu_large.py -q -x -m gpu > gpurun_out/${P}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${P}_tests.log
for c in 4 3 2; do
  timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline > gpurun_out/${P}_c$c.json 2> gpurun_out/${P}_c$c.err
done
timeout 600 python profiles/fdag_trace.py --config 4 --summary --out /tmp/t4.npz > gpurun_out/${P}_trace_c4.txt 2>&1
