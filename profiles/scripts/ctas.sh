# KKT / G_x persistent-CTA split sweep (config 2)
mkdir -p gpurun_out
for kg in ${KG:-"0 0" "3 1" "2 2" "3 2"}; do
  set -- $kg
  SGN_KKT_CTAS=$1 SGN_GX_CTAS=$2 timeout 600 python bench.py --config ${C:-2} --steps 100 --warmup 3 --no-cpu-baseline > gpurun_out/ct_$1_$2.json 2> gpurun_out/ct_$1_$2.err
  python -c "
import json
d=json.load(open('gpurun_out/ct_$1_$2.json'))
ph=d.get('phases',{})
print('kkt=$1 gx=$2', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), {k:round(v['ms'],3) for k,v in ph.items() if isinstance(v,dict) and 'ms' in v})
" 2>&1 | tail -1
done
