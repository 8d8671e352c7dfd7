#!/bin/bash
# full GPU tests with defer_groups on by default; zdist A/B
cd $GRAFT_REPO_ROOT
P=${P:-r2e}
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/${P}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${P}_tests.log
b() { timeout 600 python bench.py --config $1 --steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],2), {k:round(v['ms'],2) for k,v in d['phases'].items() if isinstance(v,dict)})"; }
for c in 4 3 2; do for Z in 2 1; do
  echo "c$c ZDIST=$Z $(SGN_ZDIST=$Z b $c)" >> gpurun_out/${P}_sweep.txt
done; done
echo "c4 ZDIST=1 ZQUOTA=128 $(SGN_ZDIST=1 SGN_ZQUOTA=128 b 4)" >> gpurun_out/${P}_sweep.txt
echo "c4 ZDIST=1 ZQUOTA=512 $(SGN_ZDIST=1 SGN_ZQUOTA=512 b 4)" >> gpurun_out/${P}_sweep.txt
SGN_ZDIST=1 timeout 600 python profiles/fdag_trace.py --config 4 --summary --out /tmp/t4.npz > gpurun_out/${P}_trace_c4_zdist1.txt 2>&1
