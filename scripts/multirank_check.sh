# Functional check of bench.py's multi-rank paths on ONE GPU (2 ranks over gloo; not a measurement)
export VP_DIST_BACKEND=gloo
for mode in sharded replicas; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
      bench.py --gpus 2 --steps 3 --warmup 3 --multi $mode --no-cpu-baseline --episodes 0 > gpurun_out/mr_$mode.log 2>&1
  echo "$mode rc=$?"; grep -c '"metric"' gpurun_out/mr_$mode.log; tail -c 400 gpurun_out/mr_$mode.log; echo
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
    bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/mr_ref.log 2>&1
echo "reference rc=$?"; grep -c '"metric"' gpurun_out/mr_ref.log; tail -c 300 gpurun_out/mr_ref.log
# the campaign harness split over 2 ranks (runs i -> rank i mod 2, records gathered to rank 0)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 \
    -m paper_2510_27191_b200 --problem tiger --iterations 4 --n-parallel 256 --particles 500 --runs 6 \
    --out gpurun_out/mr_campaign.jsonl > gpurun_out/mr_campaign.log 2>&1
echo "campaign rc=$?"; python -c "
import json; L=[json.loads(l) for l in open('gpurun_out/mr_campaign.jsonl')]
print(len(L), [l['type'] for l in L][:2], sorted(l['run_index'] for l in L if l['type']=='run'))"
