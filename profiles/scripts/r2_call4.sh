#!/bin/bash
cd $GRAFT_REPO_ROOT
P=r2i
timeout 1200 python -m pytest tests -q -m gpu -x tests/test_gpu_linear.py tests/test_gpu_sgn.py tests/test_gpu_beam.py tests/test_gpu_shell.py tests/test_gpu_large.py tests/test_gpu_batch.py tests/test_gpu_poison.py > gpurun_out/${P}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${P}_tests.log
for pair in 1 0; do
  SGN_UPD_PAIR=$pair timeout 600 python bench.py --config 4 --steps 10 --no-cpu-baseline > gpurun_out/${P}_c4_pair$pair.json 2> gpurun_out/${P}_c4_pair$pair.err
  SGN_UPD_PAIR=$pair timeout 600 python bench.py --config 2 --steps 20 --no-cpu-baseline > gpurun_out/${P}_c2_pair$pair.json 2> gpurun_out/${P}_c2_pair$pair.err
  SGN_UPD_PAIR=$pair timeout 600 python bench.py --config 3 --steps 10 --no-cpu-baseline > gpurun_out/${P}_c3_pair$pair.json 2> gpurun_out/${P}_c3_pair$pair.err
done
timeout 600 python profiles/fdag_trace.py --config 4 --summary --out /tmp/t4.npz > gpurun_out/${P}_trace_c4.txt 2>&1
