set -x
timeout 600 python -m pytest tests/test_gpu_sgn.py tests/test_gpu_poison.py tests/test_gpu_beam.py tests/test_gpu_shell.py tests/test_gpu_batch.py -x -q > gpurun_out/t2.log 2>&1; echo "exit $?" >> gpurun_out/t2.log
for G in 1 4 8; do
  for C in 2 3; do SGN_UPD_GROUP=$G timeout 300 python bench.py --config $C --steps 20 --no-cpu-baseline > gpurun_out/g${G}_c$C.json 2>/dev/null; done
  SGN_UPD_GROUP=$G timeout 300 python bench.py --config 4 --steps 5 --no-cpu-baseline > gpurun_out/g${G}_c4.json 2>/dev/null
done
