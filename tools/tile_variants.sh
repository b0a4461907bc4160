#!/bin/bash
# Build and time tile-kernel tuning variants (compile-time knobs of tile_kernels.cu) on RH and
# C3/C4.  usage: tools/tile_variants.sh "-DQCS_TILE_IO=0" "-DQCS_TILE_IO=1" ...
set -e
for v in "$@"; do
  echo "== $v"
  QCS_EXTRA_NVCC="$v" python -m paper_2411_15332_b200.build > /dev/null
  python tools/rh_timing.py 28
  python tools/time_configs.py --which c3,c4 --reps 2 | python -c 'import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d["config"], round(d["ms"],2), {k:round(x["ms"],2) for k,x in d["kernels"].items()})'
done
python -m paper_2411_15332_b200.build > /dev/null
