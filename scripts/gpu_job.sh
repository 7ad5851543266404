cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_acceptance.py -x -q -s -p no:cacheprovider > gpurun_out/acc.log 2>&1; echo "acc rc=$?"; tail -15 gpurun_out/acc.log
timeout 900 bash scripts/ncu_capture.sh r02c2 7 > gpurun_out/ncu_r02c2.log 2>&1; echo "ncu rc=$?"
