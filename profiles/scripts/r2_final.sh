#!/bin/bash
# round-2 final evidence: all GPU tests, smoke, default bench (config 4 + CPU baseline), launch list,
# ncu --set full of k_factor_dag (config 4), assembly kernel metrics (config 4)
cd $GRAFT_REPO_ROOT
P=${P:-r2fin}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${P}_smi.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu -x --durations=10 > gpurun_out/${P}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${P}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${P}_smoke.log
timeout 900 python bench.py > gpurun_out/${P}_bench_default.json 2> gpurun_out/${P}_bench_default.err
timeout 300 python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${P}_plain.json 2> gpurun_out/${P}_plain.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${P}_launches_c4.csv \
    python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${P}_ncu_launch.log 2>&1
echo "launch list rc=$?" >> gpurun_out/${P}_ncu_launch.log
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_factor_dag -c 1 \
    -o gpurun_out/${P}_fdag_c4 python profiles/profile_factor.py --config 4 > gpurun_out/${P}_ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/${P}_ncu_full.log
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv python profiles/profile_assembly.py --config 4 --reps 1 > gpurun_out/${P}_asm_ncu_c4.csv 2>&1
timeout 600 python profiles/fdag_trace.py --config 4 --summary --out /tmp/t4.npz > gpurun_out/${P}_trace_c4.txt 2>&1
for c in 2 3 1; do
  timeout 600 python bench.py --config $c --steps 20 > gpurun_out/${P}_bench_c$c.json 2> gpurun_out/${P}_bench_c$c.err
done
