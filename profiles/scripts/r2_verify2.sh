#!/bin/bash
# last verification: all GPU tests, smoke, default bench (config 4 + CPU leg), configs 2/3, solve ncu, launch list
cd $GRAFT_REPO_ROOT
P=${P:-r2v4}
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/${P}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${P}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${P}_smoke.log
timeout 900 python bench.py > gpurun_out/${P}_bench_default.json 2> gpurun_out/${P}_bench_default.err
for c in 2 3; do
  timeout 600 python bench.py --config $c --steps 20 > gpurun_out/${P}_bench_c$c.json 2> gpurun_out/${P}_bench_c$c.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${P}_launches_c4.csv \
    python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${P}_ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_solve_dag -c 1 \
    -o gpurun_out/${P}_solve_c4 python profiles/profile_factor.py --config 4 --solve > gpurun_out/${P}_ncu_solve.log 2>&1
