for L in 32 64 128 256; do for C in 2 3; do
  SGN_LEAF_SIZE=$L timeout 300 python bench.py --config $C --steps 30 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('leaf $L c$C',round(d['value'],2),d['config']['fronts'],d['config']['tree_levels'],d['config']['nnz_L'],'%.3g'%d['config']['factor_flops'],{k:round(v['ms'],3) for k,v in d['phases'].items() if isinstance(v,dict)})"
done; done
