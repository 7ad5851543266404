# search warps-per-block variants (VPB200_LIB, measurement only). Finding: 1, 2, 4 warps per block within noise at C2/C3/C5 (2 kept)
for v in base sw1 sw4 base; do for c in c2 c3 c5; do
  VPB200_LIB=variants/$v.so timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --episodes 0 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v $c', round(d['ms_per_step'],4), {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items() if k in ('search','backup')})"
done; done
