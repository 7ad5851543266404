#!/bin/bash
# A/B of the step time: this tree against a worktree of an older commit in _ab_old/ (built there).
#   bash scripts/ab_bench.sh "c2 c3 c5"
cd "$GRAFT_REPO_ROOT" || cd /root/repo
for c in ${1:-c2 c3 c5}; do
  for v in new old; do
    d=.; [ $v = old ] && d=_ab_old
    [ -d $d ] || continue
    (cd $d && timeout 300 python bench.py --config $c --no-cpu-baseline --no-secondary --episodes 0 2>/dev/null | tail -1 |
     python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d.get('kernels',{}); print('$c $v', d['ms_per_step'], d['e2e']['ms_per_step'], k.get('search',{}).get('ms_per_step'), k.get('backup',{}).get('ms_per_step'), d.get('tree_stats'))")
  done
done
