# SGN_ZQUOTA sweep on config 2 (+ factor trace at the default)
mkdir -p gpurun_out
for Q in ${QS:-0 256}; do
  for C in ${CS:-2}; do
    SGN_ZQUOTA=$Q timeout 600 python bench.py --config $C --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/zq_$Q.json 2> gpurun_out/zq_$Q.err
    python -c "
import json
d=json.load(open('gpurun_out/zq_$Q.json'))
ph=d.get('phases',{})
print('Q=$Q c$C', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), {k:round(v['ms'],3) for k,v in ph.items() if isinstance(v,dict) and 'ms' in v})
" 2>&1 | tail -1
  done
done
timeout 300 python profiles/fdag_trace.py --config 2 2>&1 | sed -n 1,20p
