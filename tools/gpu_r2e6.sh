# round 2 (session 3), call 6 (2 GPUs): new pusher (r1 loop shape + deferred block check, no extra fence, T/16 blocks): parity + A/B
set -x
export CUDA_DEVICE_MAX_CONNECTIONS=8
timeout 900 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_parity.py -q -x > gpurun_out/e6_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/e6_pytest.log
for cfg in mixtral qwen3 dsv3 dsv3_decode; do
  for kv in BASE=1 FUSCO_LIB=_ab/libs/n_minb4.so FUSCO_LIB=_ab/libs/n_fence.so FUSCO_LIB=_ab/libs/n_b128.so; do
    env $kv timeout 120 python tools/push_probe.py --config $cfg --gpus 2 --iters 15 --tag "$kv" 2>&1 | tail -1
  done
done > gpurun_out/e6_probe.jsonl
cat gpurun_out/e6_probe.jsonl
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521"
B="--steps 30 --warmup 5 --no-e2e --no-cpu-baseline"
for cfg in mixtral qwen3 dsv3 dsv3_zipf dsv3_decode; do
  for kv in BASE=1 FUSCO_LIB=_ab/libs/n_minb4.so; do
    env $kv timeout 240 $TR bench.py --gpus 2 --config $cfg $B > gpurun_out/e6_b2.json 2>gpurun_out/e6_b2.err
    python -c "import json,sys;d=json.loads([l for l in open('gpurun_out/e6_b2.json') if l.startswith('{')][-1]);print('n2 $cfg $kv',round(d['latency_us'],1),{k:round(v,1) for k,v in d['kernel_us'].items()},round(d['roofline_step_frac'],3))"
  done
done
