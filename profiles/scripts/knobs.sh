# knob sweep: config 3 (update grouping, Z quota), config 5 (leaf size)
b() { timeout 600 python bench.py --config $1 --steps ${2:-10} --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],2))"; }
for G in 8 16; do echo "c3 UPD_GROUP=$G $(SGN_UPD_GROUP=$G b 3)"; done
for Q in 64 1024; do echo "c3 ZQUOTA=$Q $(SGN_ZQUOTA=$Q b 3)"; done
for L in 32 128; do echo "c3 LEAF=$L $(SGN_LEAF_SIZE=$L b 3)"; done
for L in 64 128; do echo "c5 LEAF=$L $(SGN_LEAF_SIZE=$L timeout 600 python bench.py --config 5 --steps 5 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],2))")"; done
for G in 8 16; do echo "c5 UPD_GROUP=$G $(SGN_UPD_GROUP=$G timeout 600 python bench.py --config 5 --steps 5 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],2))")"; done
