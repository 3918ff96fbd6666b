#!/bin/bash
# ncu evidence for one bench config (1 GPU).
# Usage: bash tools/ncu_profile.sh <config> <tag> <dispatch> <combine>
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
CFG=${1:-mixtral}; TAG=${2:-r1}; D=${3:-warp}; C=${4:-warp}
mkdir -p gpurun_out
CMD="python bench.py --config $CFG --dispatch $D --combine $C --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --soak-s 0"
$CMD > gpurun_out/plain_${CFG}_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"layout_kernel|dispatch|combine" --csv --log-file gpurun_out/launches_${CFG}_${TAG}.csv $CMD \
    > gpurun_out/ncu_launch_${CFG}_${TAG}.log 2>&1
echo "launch-list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"layout_kernel|dispatch|combine" -s 30 -c 3 \
    -o gpurun_out/prof_${CFG}_${TAG} -f $CMD > gpurun_out/ncu_full_${CFG}_${TAG}.log 2>&1
echo "ncu-full rc=$?"
