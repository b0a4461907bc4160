#!/bin/bash
# A/B of planner and pass-kernel knobs on C4/C5/C3 at n=30 (tools/jit_ab.py); one process each.
cd "$(dirname "$0")/.."
run() { echo "== $1"; shift; env "$@" python tools/jit_ab.py ${CONFIGS:-c4:30 c5:30 c3:30} | python -c 'import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d["config"], d["ms"], d["sha"], d["first_s"])'; }
run jit X=1
run nosplit QCS_NO_SPLIT=1
run nodtab QCS_NO_DTAB=1
run noreal QCS_NO_REAL=1
run minb2 QCS_JIT_MINB=2
run minb4 QCS_JIT_MINB=4
run unroll2 QCS_JIT_UNROLL=2
