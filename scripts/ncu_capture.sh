# usage: bash scripts/ncu_capture.sh <tag> <kernel-regex> [skip] [count]
set -x
TAG=$1; K=$2; S=${3:-20}; C=${4:-2}
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/launches_${TAG}.csv python scripts/profile_step.py --steps 1 > /dev/null 2>&1
echo launches_rc=$?
ncu --set full --clock-control none --import-source on -k regex:${K} -s ${S} -c ${C} \
    -o gpurun_out/prof_${TAG} python scripts/profile_step.py --steps 1 > gpurun_out/ncu_${TAG}.log 2>&1
echo full_rc=$?
tail -3 gpurun_out/ncu_${TAG}.log
