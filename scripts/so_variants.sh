#!/bin/bash
# Step time of variant builds of the library (var_*.so at the repo root, timing experiments only):
#   bash scripts/so_variants.sh "v1 v2" [bench args]
cd "$GRAFT_REPO_ROOT" || cd /root/repo
cp paper_2510_27191_b200/libvpb200.so /tmp/keep_libvpb200.so
for v in base $1; do
  [ $v = base ] && cp /tmp/keep_libvpb200.so paper_2510_27191_b200/libvpb200.so || cp var_$v.so paper_2510_27191_b200/libvpb200.so
  shift 0
  timeout 300 python bench.py --no-cpu-baseline --no-secondary --episodes 0 ${@:2} 2>/dev/null | tail -1 |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d.get('kernels',{}); print('$v', d['ms_per_step'], k.get('search',{}).get('ms_per_step'), k.get('backup',{}).get('ms_per_step'))"
done
cp /tmp/keep_libvpb200.so paper_2510_27191_b200/libvpb200.so
