#!/bin/bash
# Engine A/B on all GPUs: bash tools/ab_eng.sh "<configs>" "<d:c pairs>"
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for c in $1; do
  for pr in $2; do
    d=${pr%%:*}; cm=${pr##*:}
    timeout 300 $RUN --master-port 29612 bench.py --gpus $N --config $c --dispatch $d --combine $cm --graph \
      --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/abe.log 2>&1
    echo "n=$N $c d=$d c=$cm rc=$? $(tail -1 gpurun_out/abe.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['latency_us'],1),'us',{k:round(v,1) for k,v in d['kernel_us'].items()})" 2>&1 | tail -1)"
  done
done
