# written-cell masks vs dense PSI rows (VP_DENSE_PSI=1) -- A/B of the REVERTED mask variant; kept for the record
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in c1 c2 c3 c5; do for dense in 0 1; do
  VP_DENSE_PSI=$dense timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --episodes 0 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c dense=$dense', round(d['ms_per_step'],4), d['tree_stats'], {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
done; done
