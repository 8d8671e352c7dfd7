#!/bin/bash
cd $GRAFT_REPO_ROOT
P=r2k
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/${P}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${P}_tests.log
for pair in 3 1; do
  for c in 4 2 3; do
    SGN_UPD_PAIR=$pair timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline > gpurun_out/${P}_c${c}_pair$pair.json 2> gpurun_out/${P}_c${c}_pair$pair.err
  done
done
timeout 600 python profiles/fdag_trace.py --config 4 --summary --out /tmp/t4.npz > gpurun_out/${P}_trace_c4.txt 2>&1
