#!/bin/bash
# defer_groups A/B: factor tests with the option on, bench lines both ways, config-4 trace with it on
cd $GRAFT_REPO_ROOT
P=${P:-r2d}
SGN_DEFER_GROUPS=1 timeout 900 python -m pytest tests/test_gpu_linear.py tests/test_gpu_sgn.py tests/test_gpu_large.py tests/test_gpu_batch.py -q -x -m gpu > gpurun_out/${P}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${P}_tests.log
b() { timeout 600 python bench.py --config $1 --steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],2), {k:round(v['ms'],2) for k,v in d['phases'].items() if isinstance(v,dict)})"; }
for c in 4 3 2; do for D in 0 1; do
  echo "c$c DEFER=$D $(SGN_DEFER_GROUPS=$D b $c)" >> gpurun_out/${P}_sweep.txt
done; done
SGN_DEFER_GROUPS=1 timeout 600 python profiles/fdag_trace.py --config 4 --summary --out /tmp/t4.npz > gpurun_out/${P}_trace_c4_defer.txt 2>&1
for V in "SGN_GX_FAT_TILES=2" "SGN_GX_FAT_TILES=4" "SGN_GX_LEAF_SIZE=128" "SGN_GX_LEAF_SIZE=32"; do
  echo "c4 $V $(env $V bash -c 'timeout 600 python bench.py --config 4 --steps 8 --no-cpu-baseline 2>/dev/null' | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],2), {k:round(v['ms'],2) for k,v in d['phases'].items() if isinstance(v,dict)})")" >> gpurun_out/${P}_sweep.txt
done
