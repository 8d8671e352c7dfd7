# usage: trace_kinds.sh "G list" "config list"
for G in $1; do for C in $2; do echo "== G=$G c$C"; SGN_UPD_GROUP=$G timeout 600 python profiles/fdag_trace.py --config $C --summary --out /tmp/t.npz 2>&1 | tail -9; done; done
