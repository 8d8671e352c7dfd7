b() { timeout 600 python bench.py --config 2 --steps 100 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],2), round(d['phases']['factor']['ms'],3), round(d['phases']['solve']['ms'],3))"; }
echo "default $(b)"
for Q in 64 1024; do echo "ZQUOTA=$Q $(SGN_ZQUOTA=$Q b)"; done
for L in 48 80; do echo "LEAF=$L $(SGN_LEAF_SIZE=$L b)"; done
for G in 4 1; do echo "UPD_GROUP=$G $(SGN_UPD_GROUP=$G b)"; done
