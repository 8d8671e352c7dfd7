#!/bin/bash
# G_x factorization trace (config 4) and schedule-knob sweeps on the round-2 kernel
cd $GRAFT_REPO_ROOT
P=${P:-r2k}
timeout 600 python profiles/fdag_trace.py --config 4 --which gx --summary --out /tmp/g4.npz > gpurun_out/${P}_trace_gx_c4.txt 2>&1
b() { timeout 600 python bench.py --config 4 --steps 8 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],2), {k:round(v['ms'],2) for k,v in d['phases'].items() if isinstance(v,dict)}, d['config']['fronts'], d['config']['tree_levels'])"; }
echo "default $(b)" > gpurun_out/${P}_sweep.txt
for L in 32 96 128; do echo "LEAF=$L $(SGN_LEAF_SIZE=$L b)" >> gpurun_out/${P}_sweep.txt; done
for Q in 0 64 128 512; do echo "ZQUOTA=$Q $(SGN_ZQUOTA=$Q b)" >> gpurun_out/${P}_sweep.txt; done
for T in 2 8; do echo "PAIR_MIN_TILES=$T $(SGN_PAIR_MIN_TILES=$T b)" >> gpurun_out/${P}_sweep.txt; done
for G in 16; do echo "UPD_GROUP=$G $(SGN_UPD_GROUP=$G b)" >> gpurun_out/${P}_sweep.txt; done
for G in 64; do echo "UPD_GROUP_CB=$G $(SGN_UPD_GROUP_CB=$G b)" >> gpurun_out/${P}_sweep.txt; done
for Z in 4 16; do echo "ZINLINE=$Z $(SGN_ZINLINE=$Z b)" >> gpurun_out/${P}_sweep.txt; done
