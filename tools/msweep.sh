#!/bin/bash
# Multi-GPU env sweep. Usage: bash tools/msweep.sh "<configs>" "<label|ENV=V,ENV=V>"...
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
CFGS=$1; shift
for c in $CFGS; do
  for spec in "$@"; do
    label=${spec%%|*}; envs=${spec#*|}
    env $(echo $envs | tr ',' ' ') timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus $N --config $c --steps 40 --warmup 5 --no-e2e \
      > gpurun_out/msweep_n${N}_${c}_${label}.log 2>&1
    echo "n=$N $c $label rc=$? $(tail -1 gpurun_out/msweep_n${N}_${c}_${label}.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['latency_us'],1),'us',{k:round(v,1) for k,v in d['kernel_us'].items()},'nv',{k:round(v) for k,v in d['nvlink_gbps_per_gpu'].items()})" 2>&1 | tail -1)"
  done
done
