# A/B: main tree vs _varA (same configs), traces + benches
for V in . _varA; do
  echo "==== $V"
  (cd $V && bash profiles/scripts/trace_kinds.sh "8" "2 3" 2>&1)
  (cd $V && timeout 300 python bench.py --config 2 --steps 50 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c2',d['value'],{k:round(v['ms'],3) for k,v in d['phases'].items() if isinstance(v,dict)})")
done
