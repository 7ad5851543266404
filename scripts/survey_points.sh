# SURVEY 8d measurement points beyond the default bench lines: C3 at 20 / 30 iterations,
# C4 at 65 536 rows (one JSON line each into gpurun_out/)
run() { tag=$1; shift; timeout 900 python bench.py "$@" --steps 5 --warmup 3 --no-cpu-baseline --episodes 0 2>gpurun_out/$tag.err | tail -1 > gpurun_out/$tag.json
  python -c "
import json; d=json.loads(open('gpurun_out/$tag.json').read()); print('$tag', d['ms_per_step'], round(d['value']/1e6,1), round(d['e2e']['value']/1e6,1), d['tree_stats'], {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()}, d['roofline']['frac'])" || tail -3 gpurun_out/$tag.err; }
run c3_it20 --config c3 --iterations 20
run c3_it30 --config c3 --iterations 30
run c4_n64k --config c4 --n-parallel 65536
