# usage: bash scripts/gpu_check.sh [pytest-args]   (GPU box; every step bounded by timeout)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -5 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q -x --timeout 240 -p no:cacheprovider "$@" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -40 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --cpu-budget-s 5 > gpurun_out/bench.log 2>&1; echo bench_rc=$?
tail -3 gpurun_out/bench.log
