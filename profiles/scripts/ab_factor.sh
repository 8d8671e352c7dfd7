# A/B: main tree vs _varA (same configs), traces + benches; $1 = configs to trace
for V in . _varA; do
  echo "==== $V"
  (cd $V && bash profiles/scripts/trace_kinds.sh "8" "$1" 2>&1)
  for C in $2; do
  (cd $V && timeout 300 python bench.py --config $C --steps 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c$C',d['value'],{k:round(v['ms'],3) for k,v in d['phases'].items() if isinstance(v,dict)})")
  done
done
