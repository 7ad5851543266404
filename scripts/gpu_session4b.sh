cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 300 python scripts/plugin_speed.py > gpurun_out/plugin_speed.json 2> gpurun_out/plugin_speed.err; echo "speed rc=$?"; cat gpurun_out/plugin_speed.json
timeout 600 python bench.py > gpurun_out/bench_s4.json 2> gpurun_out/bench_s4.err; echo "bench rc=$?"
