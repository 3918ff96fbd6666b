#!/bin/bash
# Quick perf matrix on 1 GPU. Usage: bash tools/gpu_perf.sh "<configs>" "<extra bench args>"
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
CFGS=${1:-mixtral}
for c in $CFGS; do
  for d in warp tma; do
    for g in "" "--graph"; do
      timeout 300 python bench.py --config $c --dispatch $d $g --steps 100 --warmup 10 --no-cpu-baseline --no-e2e $2 \
        > gpurun_out/perf_${c}_${d}${g}.log 2>&1
      echo "$c $d $g rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/perf_${c}_${d}${g}.log').read().strip().splitlines()[-1]);print(round(d['latency_us'],1),'us',{k:round(v,1) for k,v in d['kernel_us'].items()},'host',round(d['host_enqueue_ms_per_step']*1e3,1),'frac',round(d['roofline']['frac'],3))" 2>&1 | tail -1)"
    done
  done
done
