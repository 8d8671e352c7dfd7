#!/bin/bash
# config-4 per-level factor trace; G_x CTA share and update-group sweeps
cd $GRAFT_REPO_ROOT
P=${P:-r2s}
timeout 600 python profiles/fdag_trace.py --config 4 --out /tmp/t4.npz > gpurun_out/${P}_trace_c4_full.txt 2>&1
b() { timeout 600 python bench.py --config 4 --steps 8 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],2), {k:round(v['ms'],2) for k,v in d['phases'].items() if isinstance(v,dict)})"; }
echo "default $(b)" > gpurun_out/${P}_sweep.txt
for G in 56 74 111; do echo "GX_CTAS=$G $(SGN_GX_CTAS=$G b)" >> gpurun_out/${P}_sweep.txt; done
for G in 4 16; do echo "UPD_GROUP=$G $(SGN_UPD_GROUP=$G b)" >> gpurun_out/${P}_sweep.txt; done
for G in 16 64; do echo "UPD_GROUP_CB=$G $(SGN_UPD_GROUP_CB=$G b)" >> gpurun_out/${P}_sweep.txt; done
for Q in 64 1024; do echo "ZQUOTA=$Q $(SGN_ZQUOTA=$Q b)" >> gpurun_out/${P}_sweep.txt; done
