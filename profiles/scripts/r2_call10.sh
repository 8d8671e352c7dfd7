#!/bin/bash
cd $GRAFT_REPO_ROOT
P=r2o
timeout 600 python profiles/small_shell_diag.py > gpurun_out/${P}_small_shell.txt 2>&1
for c in 4 3 2; do
  timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline > gpurun_out/${P}_c$c.json 2> gpurun_out/${P}_c$c.err
done
timeout 600 python profiles/fdag_trace.py --config 4 --summary --out /tmp/t4.npz > gpurun_out/${P}_trace_c4.txt 2>&1
