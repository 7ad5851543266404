# rows per search warp sweep (VP_ROWS_PER_WARP, measurement only)
for c in c3 c5; do for r in 32 16 8; do
  VP_ROWS_PER_WARP=$r timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --episodes 0 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c rows/warp $r', round(d['ms_per_step'],4), {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
done; done
