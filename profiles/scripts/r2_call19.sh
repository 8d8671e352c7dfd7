#!/bin/bash
# ncu --set full of k_factor_dag on config 4 (current build) + G_x share sweep
cd $GRAFT_REPO_ROOT
P=${P:-r2t}
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_factor_dag -c 1 \
    -o gpurun_out/${P}_fdag_c4 python profiles/profile_factor.py --config 4 > gpurun_out/${P}_ncu_full.log 2>&1
b() { timeout 600 python bench.py --config $1 --steps 8 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],2), {k:round(v['ms'],2) for k,v in d['phases'].items() if isinstance(v,dict)})"; }
for G in 92 130 148; do echo "c4 GX_CTAS=$G $(SGN_GX_CTAS=$G b 4)" >> gpurun_out/${P}_sweep.txt; done
for G in 74 111 148; do echo "c3 GX_CTAS=$G $(SGN_GX_CTAS=$G b 3)" >> gpurun_out/${P}_sweep.txt; done
