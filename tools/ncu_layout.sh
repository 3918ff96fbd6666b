#!/bin/bash
# ncu --set full of the planner kernel (P=1) for the given configs
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for C in ${1:-dsv3_decode mixtral}; do
  CMD="python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --soak-s 0 --eager"
  $CMD > gpurun_out/plain_lay2_${C}.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"layout" -s 6 -c 1 \
      -o gpurun_out/prof_lay2_${C} -f $CMD > gpurun_out/ncu_lay2_${C}.log 2>&1
  echo "$C ncu rc=$?"
done
