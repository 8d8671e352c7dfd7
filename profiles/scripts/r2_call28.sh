#!/bin/bash
# upd_pair bit 4 (look-ahead + single-step columns as one 64x64 block below the chain rows): tests + A/B
cd $GRAFT_REPO_ROOT
P=${P:-r2g}
SGN_UPD_PAIR=31 timeout 900 python -m pytest tests/test_gpu_linear.py tests/test_gpu_sgn.py tests/test_gpu_large.py tests/test_gpu_batch.py -q -x -m gpu > gpurun_out/${P}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${P}_tests.log
b() { timeout 600 python bench.py --config $1 --steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],2), {k:round(v['ms'],2) for k,v in d['phases'].items() if isinstance(v,dict)})"; }
for c in 4 3 2; do for U in 15 31; do
  echo "c$c UPD_PAIR=$U $(SGN_UPD_PAIR=$U b $c)" >> gpurun_out/${P}_sweep.txt
done; done
SGN_UPD_PAIR=31 timeout 600 python profiles/fdag_trace.py --config 4 --summary --out /tmp/t4.npz > gpurun_out/${P}_trace_c4_pair31.txt 2>&1
