#!/bin/bash
# last verification of the committed state: all GPU tests, smoke, default bench, solve-kernel ncu
cd $GRAFT_REPO_ROOT
P=${P:-r2v2}
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/${P}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${P}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${P}_smoke.log
timeout 900 python bench.py > gpurun_out/${P}_bench_default.json 2> gpurun_out/${P}_bench_default.err
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_solve_dag -c 1 \
    -o gpurun_out/${P}_solve_c4 python profiles/profile_factor.py --config 4 --solve > gpurun_out/${P}_ncu_solve.log 2>&1
for c in 2 3; do
  timeout 600 python bench.py --config $c --steps 20 > gpurun_out/${P}_bench_c$c.json 2> gpurun_out/${P}_bench_c$c.err
done
