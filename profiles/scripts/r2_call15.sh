#!/bin/bash
cd $GRAFT_REPO_ROOT
P=r2t
timeout 1200 python bench.py --config 5 --steps 1 --warmup 1 > gpurun_out/${P}_c5.json 2> gpurun_out/${P}_c5.err
for pair in 15 7; do
  SGN_UPD_PAIR=$pair timeout 600 python bench.py --config 4 --steps 10 --no-cpu-baseline > gpurun_out/${P}_c4_pair$pair.json 2> gpurun_out/${P}_c4_pair$pair.err
done
timeout 600 python bench.py --config 3 --steps 10 --no-cpu-baseline > gpurun_out/${P}_c3.json 2> gpurun_out/${P}_c3.err
timeout 1800 python -m pytest -q -m gpu tests > gpurun_out/${P}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${P}_tests.log
timeout 600 python profiles/fdag_trace.py --config 4 --summary --out /tmp/t4.npz > gpurun_out/${P}_trace_c4.txt 2>&1
