# round 2 (session 3), call 3 (2 GPUs): push-phase A/B (poll cache, register budget, block fence), sliced TMA dispatch at P=1
set -x
export CUDA_DEVICE_MAX_CONNECTIONS=8
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "column_slices or engine_parity" > gpurun_out/e3_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/e3_pytest.log
for cfg in mixtral qwen3 dsv3 dsv3_decode; do
  for kv in BASE=1 FUSCO_FAN_POLL=1 FUSCO_LIB=_ab/libs/minb4.so FUSCO_LIB=_ab/libs/minb2.so FUSCO_LIB=_ab/libs/nofence.so FUSCO_DBG_BLK=1 FUSCO_CLAIM=token; do
    env $kv timeout 120 python tools/push_probe.py --config $cfg --gpus 2 --iters 15 --tag "$kv" 2>&1 | tail -1
  done
done > gpurun_out/e3_probe.jsonl
cat gpurun_out/e3_probe.jsonl
B1="--steps 50 --warmup 5 --no-e2e --no-cpu-baseline"
for cfg in dsv3_zipf mixtral qwen3 dsv3_decode; do
  for sl in 0 1; do
    FUSCO_TMA_SLICES=$sl timeout 200 python bench.py --config $cfg $B1 > gpurun_out/e3_n1_${cfg}_s$sl.json 2>gpurun_out/e3_n1.err
    python -c "import json,sys;d=json.loads(open('gpurun_out/e3_n1_${cfg}_s$sl.json').read().splitlines()[-1]);print('n1 $cfg slices=$sl',round(d['latency_us'],1),{k:round(v,1) for k,v in d['kernel_us'].items()},round(d['roofline_step_frac'],3))"
  done
done
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518"
B="--steps 30 --warmup 5 --no-e2e --no-cpu-baseline"
for cfg in mixtral dsv3_decode; do
  for kv in BASE=1 FUSCO_FAN_POLL=1 FUSCO_LIB=_ab/libs/minb4.so; do
    env $kv timeout 240 $TR bench.py --gpus 2 --config $cfg $B > gpurun_out/e3_b2.json 2>gpurun_out/e3_b2.err
    python -c "import json,sys;d=json.loads([l for l in open('gpurun_out/e3_b2.json') if l.startswith('{')][-1]);print('n2 $cfg $kv',round(d['latency_us'],1),{k:round(v,1) for k,v in d['kernel_us'].items()},round(d['roofline_step_frac'],3))"
  done
done
