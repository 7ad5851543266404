#!/bin/bash
# Round-2 measurement job: ncu launch lists + full captures (C2, C3), bench lines of every config,
# the launch list of the default bench command, sanitizers on small plans.
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
bash scripts/ncu_capture.sh r02c2 7 > gpurun_out/ncu_r02c2.log 2>&1
bash scripts/ncu_capture.sh r02c3 7 --n 15 --m 15 --n-parallel 65536 > gpurun_out/ncu_r02c3.log 2>&1
for c in c1 c2 c3 c4 c5; do
  timeout 600 python bench.py --config $c --no-secondary --episodes 0 $( [ $c = c2 ] || echo --no-cpu-baseline ) \
      > gpurun_out/bench_r02_$c.json 2> gpurun_out/bench_r02_$c.err
  echo "$c rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-secondary --no-cpu-baseline --episodes 0 > gpurun_out/ncu_bench.log 2>&1
echo "ncu bench rc=$?"
timeout 500 python scripts/shard_phases.py > gpurun_out/shard_c2.json 2> gpurun_out/shard_c2.err
timeout 600 python scripts/shard_phases.py --board 15 --rows-per-gpu 65536 > gpurun_out/shard_c3.json 2> gpurun_out/shard_c3.err
echo "shard rc=$?"
timeout 300 python scripts/crowdnav_step.py > gpurun_out/crowdnav_step.json 2> gpurun_out/crowdnav_step.err
echo "crowdnav rc=$?"
