mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
SGN_BICG_GRAPH=0 timeout 300 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/hostloop.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/hostloop.json')); print('hostloop c2', round(d['value'],2), d['gpu_launches'])"
export SGN_BICG_GRAPH=0
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_bench.json 2> gpurun_out/plain_bench.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_bench_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
echo "launch list rc=$?"
