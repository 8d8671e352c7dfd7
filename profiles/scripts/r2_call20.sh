#!/bin/bash
# ir_steps = 1 experiment: all GPU tests + bench lines
cd $GRAFT_REPO_ROOT
P=${P:-r2v}
export SGN_IR_STEPS=1
timeout 1800 python -m pytest tests -q -m gpu --durations=5 > gpurun_out/${P}_tests_ir1.log 2>&1
echo "rc=$?" >> gpurun_out/${P}_tests_ir1.log
for c in 4 3 2; do
  timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline > gpurun_out/${P}_ir1_c$c.json 2> gpurun_out/${P}_ir1_c$c.err
done
