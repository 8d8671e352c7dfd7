#!/bin/bash
# late hand-over of CTA slots to the G_x factorization (sgn_factor_set_retire): sweeps
cd $GRAFT_REPO_ROOT
P=${P:-r2z}
b() { timeout 600 python bench.py --config $1 --steps 8 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],2), {k:round(v['ms'],2) for k,v in d['phases'].items() if isinstance(v,dict)})"; }
timeout 300 python -m pytest tests/test_gpu_sgn.py -q -x -m gpu 2>&1 | tail -1 > gpurun_out/${P}_sweep.txt
for R in 0 4 8 16; do for G in 111 185; do
  echo "c4 RETIRE=$R GX_CTAS=$G $(SGN_GX_RETIRE=$R SGN_GX_CTAS=$G b 4)" >> gpurun_out/${P}_sweep.txt
done; done
echo "c4 RETIRE=8 GX_CTAS=296 $(SGN_GX_RETIRE=8 SGN_GX_CTAS=296 b 4)" >> gpurun_out/${P}_sweep.txt
for R in 0 4 8; do
  echo "c3 RETIRE=$R $(SGN_GX_RETIRE=$R b 3)" >> gpurun_out/${P}_sweep.txt
  echo "c2 RETIRE=$R $(SGN_GX_RETIRE=$R b 2)" >> gpurun_out/${P}_sweep.txt
done
