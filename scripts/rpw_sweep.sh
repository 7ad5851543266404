# leaves per backup warp sweep (VP_LEAVES_PER_WARP, measurement only) on the bench configs
for c in c2 c3 c5; do
for l in 32 16 8 6 4 2; do
  VP_LEAVES_PER_WARP=$l timeout 300 python bench.py --config $c --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c lpw $l', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']/1e6,1))"
done; done
