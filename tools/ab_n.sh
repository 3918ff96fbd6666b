#!/bin/bash
# A/B of env settings on the multi-GPU bench: bash tools/ab_n.sh "<configs>" "<envA>" "<envB>" ...
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
cfgs=$1; shift
for c in $cfgs; do
  for envs in "$@"; do
    env $envs timeout 300 $RUN --master-port 29611 bench.py --gpus $N --config $c --graph --steps 50 --warmup 5 \
      --no-e2e --no-cpu-baseline > gpurun_out/ab.log 2>&1
    echo "n=$N $c [$envs] rc=$? $(tail -1 gpurun_out/ab.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['latency_us'],1),'us',{k:round(v,1) for k,v in d['kernel_us'].items()})" 2>&1 | tail -1)"
  done
done
