#!/bin/bash
# Quick perf matrix on 1 GPU. Usage: bash tools/gpu_perf.sh "<configs>" "<engine pairs d:c>" "<extra bench args>"
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
CFGS=${1:-mixtral}
PAIRS=${2:-"warp:warp tma:tma"}
for c in $CFGS; do
  for pr in $PAIRS; do
    d=${pr%%:*}; cm=${pr##*:}
    timeout 300 python bench.py --config $c --dispatch $d --combine $cm --graph --steps 100 --warmup 10 \
      --no-cpu-baseline --no-e2e $3 > gpurun_out/perf_${c}_${d}_${cm}.log 2>&1
    echo "$c d=$d c=$cm rc=$? $(python -c "import json,sys;d=json.loads(open('gpurun_out/perf_${c}_${d}_${cm}.log').read().strip().splitlines()[-1]);print(round(d['latency_us'],1),'us',{k:round(v,1) for k,v in d['kernel_us'].items()},'tmin',{k:round(v,1) for k,v in d['t_min_us'].items()},'frac',round(d['roofline']['frac'],3))" 2>&1 | tail -1)"
  done
done
