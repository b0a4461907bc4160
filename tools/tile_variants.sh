#!/bin/bash
# Build and time the tile-kernel tuning variants (QCS_TILE_NG / QCS_TILE_MINB) on C3/C4.
set -e
mkdir -p gpurun_out
for v in "-DQCS_TILE_NG=1 -DQCS_TILE_MINB=2" "-DQCS_TILE_NG=2 -DQCS_TILE_MINB=1" "-DQCS_TILE_NG=1 -DQCS_TILE_MINB=1" "-DQCS_TILE_NG=2 -DQCS_TILE_MINB=2"; do
  echo "== $v"
  QCS_EXTRA_NVCC="$v" python -m paper_2411_15332_b200.build > /dev/null
  python tools/time_configs.py --which c3,c4 --reps 2 | python -c 'import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d["config"], round(d["ms"],2), {k:round(x["ms"],2) for k,x in d["kernels"].items()})'
done
python -m paper_2411_15332_b200.build > /dev/null
