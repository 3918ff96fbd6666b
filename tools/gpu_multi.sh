#!/bin/bash
# Multi-GPU validation + bench on all GPUs of the box. Usage: bash tools/gpu_multi.sh [configs]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
for d in warp tma; do
  FUSCO_DISPATCH=$d timeout 600 python -m pytest tests/test_gpu_multiproc.py -q -rf > gpurun_out/mp_${d}.log 2>&1
  echo "multiproc $d rc=$?"; tail -3 gpurun_out/mp_${d}.log
done
for c in ${1:-mixtral}; do
  for d in warp tma; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
      bench.py --gpus $N --config $c --dispatch $d --steps 50 --warmup 5 --no-e2e > gpurun_out/bench_n${N}_${c}_${d}.log 2>&1
    echo "bench n=$N $c $d rc=$?"
    tail -1 gpurun_out/bench_n${N}_${c}_${d}.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['latency_us'],1),'us',{k:round(v,1) for k,v in d['kernel_us'].items()},'t_min',{k:round(v,1) for k,v in d['t_min_us'].items()},'frac',round(d['roofline']['frac'],3), d['nvlink_gbps_per_gpu'])" 2>&1 | tail -1
  done
done
