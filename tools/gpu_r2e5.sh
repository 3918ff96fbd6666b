# round 2 (session 3), call 5 (2 GPUs): which part of the P>1 pusher costs the throughput (compile-time variants)
set -x
export CUDA_DEVICE_MAX_CONNECTIONS=8
for cfg in mixtral dsv3; do
  for kv in BASE=1 FUSCO_LIB=_ab/libs/pushr1.so FUSCO_LIB=_ab/libs/pushr1_b512.so FUSCO_LIB=_ab/libs/b512.so FUSCO_LIB=_ab/libs/pushr1_nofence.so "FUSCO_DISPATCH=tma" "FUSCO_LIB=_ab/libs/pushr1.so FUSCO_NODEDUP=1"; do
    env $kv timeout 120 python tools/push_probe.py --config $cfg --gpus 2 --iters 15 --tag "$kv" 2>&1 | tail -1
  done
  for kv in BASE=1 FUSCO_LIB=_ab/libs/pushr1.so FUSCO_LIB=_ab/libs/pushr1_nob.so; do
    env $kv timeout 120 python tools/push_probe.py --config $cfg --gpus 2 --iters 15 --push-only --tag "pushonly $kv" 2>&1 | tail -1
  done
done > gpurun_out/e5_probe.jsonl
cat gpurun_out/e5_probe.jsonl
timeout 120 python tools/hbm_probe.py > gpurun_out/e5_hbm.json 2>&1; cat gpurun_out/e5_hbm.json
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29520"
B="--steps 30 --warmup 5 --no-e2e --no-cpu-baseline"
for cfg in mixtral dsv3 dsv3_decode; do
  for kv in FUSCO_LIB=_ab/libs/pushr1.so FUSCO_LIB=_ab/libs/pushr1_b512.so FUSCO_LIB=_ab/libs/b512.so; do
    env $kv timeout 240 $TR bench.py --gpus 2 --config $cfg $B > gpurun_out/e5_b2.json 2>gpurun_out/e5_b2.err
    python -c "import json,sys;d=json.loads([l for l in open('gpurun_out/e5_b2.json') if l.startswith('{')][-1]);print('n2 $cfg $kv',round(d['latency_us'],1),{k:round(v,1) for k,v in d['kernel_us'].items()},round(d['roofline_step_frac'],3))"
  done
done
