# warp-level aggregation of sibling action deliveries in k_backup -- A/B of a REVERTED variant: no measurable effect (siblings rarely share a backup warp)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in noagg agg noagg agg; do for c in c2 c3 c5; do
  VPB200_LIB=variants/$v.so timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --episodes 0 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v $c', round(d['ms_per_step'],4), {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items() if k in ('search','backup')})"
done; done
