#!/bin/bash
# Multi-GPU validation + probe + bench on all GPUs of the box.
# Usage: bash tools/gpu_multi.sh "<configs>" "<engine pairs d:c>" [extra env]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 300 $RUN --master-port 29501 tools/p2p_probe.py 256 > gpurun_out/p2p_n${N}.log 2>&1
echo "p2p n=$N rc=$? $(tail -1 gpurun_out/p2p_n${N}.log)"
if [ -z "$SKIP_MP" ]; then
  FUSCO_DISPATCH=tma FUSCO_COMBINE=tma timeout 600 python -m pytest tests/test_gpu_multiproc.py -q -rf > gpurun_out/mp_tma.log 2>&1
  echo "multiproc tma rc=$?"; tail -2 gpurun_out/mp_tma.log
fi
for c in ${1:-mixtral}; do
  for pr in ${2:-"warp:warp tma:tma"}; do
    d=${pr%%:*}; cm=${pr##*:}
    timeout 600 $RUN --master-port 29511 bench.py --gpus $N --config $c --dispatch $d --combine $cm --graph \
      --steps 50 --warmup 5 --no-e2e > gpurun_out/bench_n${N}_${c}_${d}_${cm}.log 2>&1
    echo "bench n=$N $c d=$d c=$cm rc=$? $(tail -1 gpurun_out/bench_n${N}_${c}_${d}_${cm}.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['latency_us'],1),'us',{k:round(v,1) for k,v in d['kernel_us'].items()},'t_min',{k:round(v,1) for k,v in d['t_min_us'].items()},'frac',round(d['roofline']['frac'],3), d['nvlink_gbps_per_gpu'])" 2>&1 | tail -1)"
  done
done
