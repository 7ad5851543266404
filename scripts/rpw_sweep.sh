# rows per search warp / leaves per backup warp sweeps (VP_ROWS_PER_WARP / VP_LEAVES_PER_WARP, measurement only)
for c in c1 c2; do for r in 32 16 8 4; do
  VP_ROWS_PER_WARP=$r timeout 300 python bench.py --config $c --steps 20 --warmup 5 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c rows/warp $r', round(d['ms_per_step'],4), {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
done; done
