for rep in 1 2 3; do for e in 0 1; do
QCS_POOL_KEEP=$e timeout 300 python bench.py --workload c1 --steps 20 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c1 keep=$e', round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), d['e2e'].get('mode'), round(d['e2e'].get('serial_ms_per_step',0),3))"
done; done
