mkdir -p gpurun_out
timeout 1100 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for C in 2 3 5; do
  timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/sw_c$C.json 2> gpurun_out/sw_c$C.err
  python -c "
import json
d=json.load(open('gpurun_out/sw_c$C.json'))
ph=d.get('phases',{})
print('c$C', round(d['value'],2), 'ms', round(d['ms_per_step'],3), {k:(round(v['ms'],3)) for k,v in ph.items() if isinstance(v,dict) and 'ms' in v})
" 2>&1 | tail -1
done
timeout 900 python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/sw_c4.json 2> gpurun_out/sw_c4.err
python -c "
import json
d=json.load(open('gpurun_out/sw_c4.json'))
ph=d.get('phases',{})
print('c4', round(d['value'],3), 'ms', round(d['ms_per_step'],3), {k:(round(v['ms'],3)) for k,v in ph.items() if isinstance(v,dict) and 'ms' in v}, 'tflops', round(d['roofline']['achieved'],2))
" 2>&1 | tail -1
