#!/bin/bash
# round-2 re-entry cycle: all GPU tests, default bench (config 4 + CPU baseline), the config-4 ncu launch
# list, ncu --set full of k_factor_dag / k_solve_dag (config 4), compute-sanitizer on smoke()
cd $GRAFT_REPO_ROOT
P=${P:-r2q}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${P}_smi.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu -x --durations=25 > gpurun_out/${P}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${P}_tests.log
timeout 900 python bench.py > gpurun_out/${P}_bench_default.json 2> gpurun_out/${P}_bench_default.err
timeout 300 python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${P}_plain.json 2> gpurun_out/${P}_plain.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${P}_launches_c4.csv \
    python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${P}_ncu_launch.log 2>&1
echo "launch list rc=$?" >> gpurun_out/${P}_ncu_launch.log
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_factor_dag -c 1 \
    -o gpurun_out/${P}_fdag_c4 python profiles/profile_factor.py --config 4 > gpurun_out/${P}_ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/${P}_ncu_full.log
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_solve_dag -c 1 \
    -o gpurun_out/${P}_solve_c4 python profiles/profile_factor.py --config 4 --solve > gpurun_out/${P}_ncu_solve.log 2>&1
echo "ncu solve rc=$?" >> gpurun_out/${P}_ncu_solve.log
timeout 600 compute-sanitizer --tool memcheck --leak-check no python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_memcheck.txt 2>&1
echo "memcheck rc=$?" >> gpurun_out/${P}_memcheck.txt
timeout 600 compute-sanitizer --tool synccheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_synccheck.txt 2>&1
echo "synccheck rc=$?" >> gpurun_out/${P}_synccheck.txt
