#!/bin/bash
cd $GRAFT_REPO_ROOT
P=r2l
timeout 900 python -m pytest -q tests/test_gpu_poison.py tests/test_gpu_shell.py tests/test_gpu_linear.py tests/test_gpu_sgn.py tests/test_gpu_large.py > gpurun_out/${P}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${P}_tests.log
for pair in 7 3; do
  for c in 4 2; do
    SGN_UPD_PAIR=$pair timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline > gpurun_out/${P}_c${c}_pair$pair.json 2> gpurun_out/${P}_c${c}_pair$pair.err
  done
done
timeout 600 python profiles/fdag_trace.py --config 4 --summary --out /tmp/t4.npz > gpurun_out/${P}_trace_c4.txt 2>&1
timeout 900 python profiles/c4_parity_diag.py > gpurun_out/${P}_c4diag.txt 2>&1
