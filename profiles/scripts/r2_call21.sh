#!/bin/bash
# shell kernel specialisation check: shell tests, config-4 bench, assembly kernel times
cd $GRAFT_REPO_ROOT
P=${P:-r2w}
timeout 900 python -m pytest tests/test_gpu_shell.py -q -x -m gpu > gpurun_out/${P}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${P}_tests.log
timeout 600 python bench.py --config 4 --steps 10 --no-cpu-baseline > gpurun_out/${P}_c4.json 2> gpurun_out/${P}_c4.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv python profiles/profile_assembly.py --config 4 --reps 1 > gpurun_out/${P}_asm_ncu_c4.csv 2>&1
