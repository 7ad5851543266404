# usage: bash scripts/ncu_capture.sh <tag> [skip] [extra profile_step args]
# 1. launch list of one planning step with per-launch duration and DRAM bytes (roofline traffic)
# 2. full captures of k_search and k_backup (launch index `skip` = pass skip+1, default pass 8)
set -x
TAG=$1; S=${2:-7}; shift; shift
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/launches_${TAG}.csv python scripts/profile_step.py --steps 1 "$@" > /dev/null 2>&1
echo launches_rc=$?
for K in k_search k_backup; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:${K} -s ${S} -c 1 \
      -o gpurun_out/prof_${TAG}_${K} python scripts/profile_step.py --steps 1 "$@" > gpurun_out/ncu_${TAG}_${K}.log 2>&1
  echo ${K}_rc=$?
  tail -2 gpurun_out/ncu_${TAG}_${K}.log
done
