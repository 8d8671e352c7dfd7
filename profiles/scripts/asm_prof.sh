timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "exit $?" >> gpurun_out/gputests.log
for C in $1; do
  timeout 300 python profiles/profile_assembly.py --config $C --reps 1 > gpurun_out/asm_c$C.log 2>&1
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv python profiles/profile_assembly.py --config $C --reps 1 > gpurun_out/asm_ncu_c$C.csv 2>&1
done
timeout 300 python bench.py --config 5 --steps 20 > gpurun_out/bench_c5.json 2>gpurun_out/bench_c5.err
