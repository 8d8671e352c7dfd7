# G_x persistent-CTA share sweep (config 2); the KKT factor gets the rest of SMs x 4
mkdir -p gpurun_out
for g in ${GS:-148 74 37 222}; do
  SGN_GX_CTAS=$g timeout 600 python bench.py --config ${C:-2} --steps 100 --warmup 3 --no-cpu-baseline > gpurun_out/ct_$g.json 2> gpurun_out/ct_$g.err
  python -c "
import json
d=json.load(open('gpurun_out/ct_$g.json'))
ph=d.get('phases',{})
print('gx=$g', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), {k:round(v['ms'],3) for k,v in ph.items() if isinstance(v,dict) and 'ms' in v})
" 2>&1 | tail -1
done
