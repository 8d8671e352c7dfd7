#!/bin/bash
# G_x share re-sweep on the final kernel (configs 4, 3)
cd $GRAFT_REPO_ROOT
P=${P:-r2h}
b() { timeout 600 python bench.py --config $1 --steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],2), {k:round(v['ms'],2) for k,v in d['phases'].items() if isinstance(v,dict)})"; }
for G in 100 111 120 130 140; do echo "c4 GX_CTAS=$G $(SGN_GX_CTAS=$G b 4)" >> gpurun_out/${P}_sweep.txt; done
for G in 100 111 130; do echo "c3 GX_CTAS=$G $(SGN_GX_CTAS=$G b 3)" >> gpurun_out/${P}_sweep.txt; done
