mkdir -p gpurun_out
for C in 1 2 3 5; do
  timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/sw_c$C.json 2> gpurun_out/sw_c$C.err
  echo "c$C rc=$?"
done
timeout 900 python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/sw_c4.json 2> gpurun_out/sw_c4.err; echo "c4 rc=$?"
timeout 300 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/sw_ref.json 2> gpurun_out/sw_ref.err; echo "ref rc=$?"
for C in 1 2 3 4 5; do python -c "
import json,sys
d=json.load(open('gpurun_out/sw_c$C.json'))
ph=d.get('phases',{})
print('c$C', round(d['value'],2), d['unit'], 'ms', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value'],2) if d.get('e2e') else None, {k:(round(v['ms'],3) if isinstance(v,dict) and 'ms' in v else None) for k,v in ph.items() if isinstance(v,dict)}, 'roof', round(d['roofline']['frac'],4) if d.get('roofline') else None)
" 2>&1 | tail -1; done
cat gpurun_out/sw_ref.json | head -c 600
