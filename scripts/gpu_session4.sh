cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_philox.py tests/test_gpu_plugin.py -q > gpurun_out/new_tests.log 2>&1; echo "new rc=$?"
bash scripts/ab_bench.sh "c2 c3" > gpurun_out/ab_tmpl.txt 2>&1; bash scripts/ab_bench.sh "c2" >> gpurun_out/ab_tmpl.txt 2>&1; cat gpurun_out/ab_tmpl.txt
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_r2s4.log 2>&1; echo "full rc=$?"; tail -3 gpurun_out/gputest_r2s4.log
