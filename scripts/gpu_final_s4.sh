#!/bin/bash
# Final measurement pass of the round-2 build (Philox / plug-ins): GPU tests, smoke, the default
# bench line, the launch list of the default bench command, full ncu captures of k_search /
# k_backup at C2 and their traffic.
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/final_gputest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/final_gputest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-secondary --no-cpu-baseline --episodes 0 > gpurun_out/final_ncu_bench.log 2>&1
echo "ncu bench rc=$?"
bash scripts/ncu_capture.sh finalc2 7 > gpurun_out/ncu_finalc2.log 2>&1; echo "capture rc=$?"
