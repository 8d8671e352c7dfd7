#!/bin/bash
cd $GRAFT_REPO_ROOT
P=r2m
timeout 900 python -m pytest -q tests/test_gpu_poison.py tests/test_gpu_shell.py tests/test_gpu_linear.py tests/test_gpu_sgn.py tests/test_gpu_large.py tests/test_gpu_minimize_batched.py tests/test_gpu_lbfgs.py > gpurun_out/${P}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${P}_tests.log
for g in 16 8; do
  SGN_UPD_GROUP=$g timeout 600 python bench.py --config 4 --steps 10 --no-cpu-baseline > gpurun_out/${P}_c4_g$g.json 2> gpurun_out/${P}_c4_g$g.err
done
timeout 600 python bench.py --config 2 --steps 20 --no-cpu-baseline > gpurun_out/${P}_c2.json 2> gpurun_out/${P}_c2.err
export SGN_BICG_GRAPH=0
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_factor_dag -s 2 -c 1 \
    -o gpurun_out/${P}_fdag_c4 python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${P}_ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/${P}_ncu_full.log
