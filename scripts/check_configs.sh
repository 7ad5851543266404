timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in c1 c2 c3 c5; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"; done
