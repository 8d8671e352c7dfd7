# repeat the c2 bench R times (variance check) + one factor trace
mkdir -p gpurun_out
for r in $(seq 1 ${R:-3}); do
  timeout 600 python bench.py --config ${C:-2} --steps 100 --warmup 3 --no-cpu-baseline > gpurun_out/rep_$r.json 2> gpurun_out/rep_$r.err
  python -c "
import json
d=json.load(open('gpurun_out/rep_$r.json'))
ph=d.get('phases',{})
print('rep $r', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), d['clocks'].get('sm_mhz'), {k:round(v['ms'],3) for k,v in ph.items() if isinstance(v,dict) and 'ms' in v})
" 2>&1 | tail -1
done
