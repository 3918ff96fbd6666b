#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for L in grid cluster; do
  for C in mixtral dsv3_decode; do
    CMD="python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --soak-s 0 --eager"
    FUSCO_LAYOUT=$L $CMD > gpurun_out/plain_lay_${L}_${C}.log 2>&1 && \
    FUSCO_LAYOUT=$L ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 \
        -k regex:"layout" -s 6 -c 2 -o gpurun_out/prof_layout_${L}_${C} -f $CMD > gpurun_out/ncu_lay_${L}_${C}.log 2>&1
    echo "$L $C ncu rc=$?"
    FUSCO_LAYOUT=$L FUSCO_TRACE=1 python tools/trace_step.py $C > gpurun_out/trace_${L}_${C}.log 2>&1
    cat gpurun_out/trace_${L}_${C}.log | tail -14
  done
done
