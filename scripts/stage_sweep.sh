# per-warp TMA stage budget sweep (VP_STAGE_KB, measurement only)
for c in c2 c3 c5; do for kb in 2 4 8 16 32; do
  VP_STAGE_KB=$kb timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --episodes 0 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c stage_kb $kb', round(d['ms_per_step'],4), {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
done; done
