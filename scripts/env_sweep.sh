#!/bin/bash
# Step time under an environment override (measurement only):  bash scripts/env_sweep.sh VAR "v1 v2" "c2 c3"
cd "$GRAFT_REPO_ROOT" || cd /root/repo
for c in $3; do for v in $2; do
  env $1=$v timeout 300 python bench.py --config $c --no-cpu-baseline --no-secondary --episodes 0 2>/dev/null | tail -1 |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d.get('kernels',{}); print('$c $1=$v', d['ms_per_step'], d['e2e']['ms_per_step'], k.get('search',{}).get('ms_per_step'), k.get('backup',{}).get('ms_per_step'), d['tree_stats'])"
done; done
