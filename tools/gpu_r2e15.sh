# round 2 (session 3), call 15 (2 GPUs): owner-side pre-reduction: parity (emulated + multi-process), A/B benches
set -x
export FUSCO_BENCH_WATCHDOG_S=150
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "owner_reduce or engine_parity or bf16_parity or fp32" > gpurun_out/e15_pytest1.log 2>&1; echo pytest1_rc=$?; tail -15 gpurun_out/e15_pytest1.log
timeout 1200 python -m pytest tests/test_gpu_multiproc.py -q -x > gpurun_out/e15_pytest2.log 2>&1; echo pytest2_rc=$?; tail -15 gpurun_out/e15_pytest2.log
summ() { python - "$1" "$2" <<'PY'
import json,sys
f=sys.argv[1]
try:
    d=json.loads([l for l in open(f) if l.startswith('{"metric"')][-1])
    print(sys.argv[2], round(d['latency_us'],1), {k:round(v,1) for k,v in d['kernel_us'].items()}, round(d['roofline_step_frac'],3), d.get('owner_reduce'))
except Exception as e: print(sys.argv[2], 'ERR', e)
PY
}
B="--steps 30 --warmup 5 --no-e2e --no-cpu-baseline"
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29680"
for cfg in dsv3 dsv3_zipf qwen3 dsv3_decode mixtral; do
  for kv in BASE=1 FUSCO_OWNER_REDUCE=0; do
    env $kv timeout 240 $TR bench.py --gpus 2 --config $cfg $B > gpurun_out/e15_b2.json 2> gpurun_out/e15_b2.err; summ gpurun_out/e15_b2.json "n2 $cfg $kv"
  done
done
tail -5 gpurun_out/e15_b2.err
