#!/bin/bash
# round-2 profile of config 4: factorization task trace, ncu launch list, ncu --set full of
# k_factor_dag, and compute-sanitizer memcheck/synccheck of the persistent kernels on config 1
cd $GRAFT_REPO_ROOT
P=${P:-r2p}
timeout 600 python profiles/fdag_trace.py --config 4 --summary --out /tmp/t4.npz > gpurun_out/${P}_trace_c4.txt 2>&1
timeout 600 python profiles/fdag_trace.py --config 2 --summary --out /tmp/t2.npz > gpurun_out/${P}_trace_c2.txt 2>&1
export SGN_BICG_GRAPH=0
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${P}_launches_c4.csv \
    python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${P}_ncu_launch.log 2>&1
echo "launch list rc=$?" >> gpurun_out/${P}_ncu_launch.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_factor_dag -s 2 -c 1 \
    -o gpurun_out/${P}_fdag_c4 python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${P}_ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/${P}_ncu_full.log
unset SGN_BICG_GRAPH
timeout 900 compute-sanitizer --tool memcheck --leak-check no python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_memcheck.txt 2>&1
echo "memcheck rc=$?" >> gpurun_out/${P}_memcheck.txt
timeout 900 compute-sanitizer --tool synccheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_synccheck.txt 2>&1
echo "synccheck rc=$?" >> gpurun_out/${P}_synccheck.txt
