#!/bin/bash
cd $GRAFT_REPO_ROOT
P=r2n
timeout 1500 python -m pytest -q -m gpu tests > gpurun_out/${P}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${P}_tests.log
for cb in 32 8 72; do
  SGN_UPD_GROUP_CB=$cb timeout 600 python bench.py --config 4 --steps 10 --no-cpu-baseline > gpurun_out/${P}_c4_cb$cb.json 2> gpurun_out/${P}_c4_cb$cb.err
done
timeout 600 python bench.py --config 2 --steps 20 --no-cpu-baseline > gpurun_out/${P}_c2.json 2> gpurun_out/${P}_c2.err
timeout 600 python bench.py --config 3 --steps 10 --no-cpu-baseline > gpurun_out/${P}_c3.json 2> gpurun_out/${P}_c3.err
timeout 600 python profiles/fdag_trace.py --config 4 --summary --out /tmp/t4.npz > gpurun_out/${P}_trace_c4.txt 2>&1
