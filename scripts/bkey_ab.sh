# belief-key mode A/B (VP_BKEY_MODE=0: (action row, obs) keys, claims in sequence; 1: (belief, action, obs),
# both claims of a level in flight together) -- measurement only
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for m in 0 1 0 1; do for c in c2 c3 c5; do
  VP_BKEY_MODE=$m timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --episodes 0 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('mode$m $c', round(d['ms_per_step'],4), d['tree_stats'], {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items() if k in ('search','backup')})"
done; done
