mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pt.txt
for C in 1 2; do
  timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/q_c$C.json 2> gpurun_out/q_c$C.err
  python -c "
import json
d=json.load(open('gpurun_out/q_c$C.json'))
ph=d.get('phases',{})
print('c$C', round(d['value'],2), 'ms', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value'],2), {k:(round(v['ms'],3), v.get('bicgstab_iters')) for k,v in ph.items() if isinstance(v,dict) and 'ms' in v}, 'launches', d['gpu_launches'])
" 2>&1 | tail -1
done
cat gpurun_out/pt.txt
