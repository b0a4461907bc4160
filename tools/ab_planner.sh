cd /root/repo
run() { echo "== $1"; shift; env "$@" python tools/time_configs.py --which c4,c5 --n4 30 --n5 30 --reps 3 | python -c 'import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d["config"], round(d["ms"],2), round(d["norm"],12))'; }
run old QCS_B200_LIB=paper_2411_15332_b200/libqcs_old.so
run new X=1
run nosplit QCS_NO_SPLIT=1
run nodtab QCS_NO_DTAB=1
run noreal QCS_NO_REAL=1
run nodtab_noreal QCS_NO_DTAB=1 QCS_NO_REAL=1
