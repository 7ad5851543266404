# backup block shape variants (VPB200_LIB, measurement only). Finding: an explicit __launch_bounds__(256, 1) lets k_backup take 165 registers (8 warps/SM, -6%); the committed build (128 regs, 16 warps/SM) equals the best variant (16-warp blocks)
for v in bw16 bw8m3 base bw16 base; do for c in c2 c3 c5; do
  VPB200_LIB=variants/$v.so timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --episodes 0 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v $c', round(d['ms_per_step'],4), {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items() if k in ('search','backup')})"
done; done
