#!/bin/bash
cd $GRAFT_REPO_ROOT
P=${P:-r2m}
timeout 900 python -m pytest tests/test_gpu_linear.py tests/test_gpu_sgn.py tests/test_gpu_large.py tests/test_gpu_batch.py tests/test_gpu_dgn.py -q -x -m gpu > gpurun_out/${P}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${P}_tests.log
for c in 4 3 2; do
  timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c$c', round(d['value'],2), {k:round(v['ms'],3) for k,v in d['phases'].items() if isinstance(v,dict)})" >> gpurun_out/${P}_sweep.txt
done
