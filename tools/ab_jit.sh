#!/bin/bash
# A/B of planner and pass-kernel knobs on C4/C5/C3 at n=30 (tools/jit_ab.py); one process each.
# usage: tools/ab_jit.sh "name ENV=val ..." ...   (default: the set below)
cd "$(dirname "$0")/.."
run() { local name=$1; shift; echo "== $name"; env "$@" python tools/jit_ab.py ${CONFIGS:-c4:30 c5:30 c3:30} | python -c 'import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d["config"], d["ms"], d["sha"], d["first_s"])'; }
if [ $# -eq 0 ]; then
  set -- "default X=1" "nobankswap QCS_JIT_BANKSWAP=0" "interpreter QCS_JIT=0"
fi
for v in "$@"; do run $v; done
