#!/bin/bash
# round-2 measurement cycle: bench lines for configs 2, 3, 5, the reference arm (config 4),
# the config-4 ncu launch list and ncu --set full of k_factor_dag / k_solve_dag on config 4
cd $GRAFT_REPO_ROOT
P=${P:-r2m}
timeout 600 python bench.py --config 2 --steps 20 > gpurun_out/${P}_bench_c2.json 2> gpurun_out/${P}_bench_c2.err
timeout 600 python bench.py --config 3 --steps 10 > gpurun_out/${P}_bench_c3.json 2> gpurun_out/${P}_bench_c3.err
timeout 900 python bench.py --config 5 --steps 2 --warmup 1 > gpurun_out/${P}_bench_c5.json 2> gpurun_out/${P}_bench_c5.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/${P}_bench_ref.json 2> gpurun_out/${P}_bench_ref.err
nproc > gpurun_out/${P}_nproc.txt
export SGN_BICG_GRAPH=0
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${P}_launches_c4.csv \
    python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${P}_ncu_launch.log 2>&1
echo "launch list rc=$?" >> gpurun_out/${P}_ncu_launch.log
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_factor_dag -c 1 \
    -o gpurun_out/${P}_fdag_c4 python profiles/profile_factor.py --config 4 > gpurun_out/${P}_ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/${P}_ncu_full.log
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_solve_dag -c 1 \
    -o gpurun_out/${P}_solve_c4 python profiles/profile_factor.py --config 4 --solve > gpurun_out/${P}_ncu_solve.log 2>&1
echo "ncu solve rc=$?" >> gpurun_out/${P}_ncu_solve.log
