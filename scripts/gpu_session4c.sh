cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_philox.py tests/test_gpu_kernels.py tests/test_gpu_sir.py tests/test_gpu_plan.py -q -x > gpurun_out/pair_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pair_tests.log
for r in splitmix64 philox; do timeout 300 python scripts/crowdnav_step.py --rng $r > gpurun_out/crowd_$r.json 2>gpurun_out/crowd_$r.err; echo "crowd $r rc=$?"; done
for c in c4; do for r in splitmix64 philox; do timeout 300 python bench.py --config $c --rng $r --no-cpu-baseline --no-secondary --episodes 0 > gpurun_out/bench_${c}_$r.json 2>/dev/null; echo "$c $r rc=$?"; done; done
python - <<'P'
import json
for r in ("splitmix64","philox"):
    d=json.load(open(f"gpurun_out/crowd_{r}.json")); print("crowdnav", r, round(d["ms_per_step"],3), {k: round(v,3) for k,v in d["kernel_ms_per_step"].items()})
    d=json.loads(open(f"gpurun_out/bench_c4_{r}.json").read().strip().splitlines()[-1]); print("c4", r, d["ms_per_step"], d["kernels"]["search"]["ms_per_step"] if "search" in d.get("kernels",{}) else "")
P
