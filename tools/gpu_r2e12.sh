# round 2 (session 3), call 12 (2 GPUs): per-CTA-round completion counting vs per-unit: parity, push probe, benches
set -x
export FUSCO_BENCH_WATCHDOG_S=150
timeout 1200 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_parity.py -q -x > gpurun_out/e12_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/e12_pytest.log
for cfg in mixtral dsv3 qwen3 dsv3_decode; do
  for kv in BASE=1 FUSCO_PUSH_ROUNDS=0 FUSCO_BALANCE=0; do
    env $kv timeout 120 python tools/push_probe.py --config $cfg --gpus 2 --iters 15 --tag "$kv" 2>&1 | tail -1
  done
done > gpurun_out/e12_probe.jsonl
python - <<'PY'
import json
for l in open('gpurun_out/e12_probe.jsonl'):
    if not l.startswith('{'): print(l.strip()[:200]); continue
    d=json.loads(l); print(d['config'], d['tag'][:30].ljust(30), d['us'], 'push', d['push_gbps'])
PY
summ() { python - "$1" "$2" <<'PY'
import json,sys
f=sys.argv[1]
try:
    d=json.loads([l for l in open(f) if l.startswith('{"metric"')][-1])
    print(sys.argv[2], round(d['latency_us'],1), {k:round(v,1) for k,v in d['kernel_us'].items()}, round(d['roofline_step_frac'],3))
except Exception as e: print(sys.argv[2], 'ERR', e)
PY
}
B="--steps 30 --warmup 5 --no-e2e --no-cpu-baseline"
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29660"
for cfg in mixtral dsv3 dsv3_zipf qwen3 dsv3_decode; do
  for kv in BASE=1 FUSCO_PUSH_ROUNDS=0; do
    env $kv timeout 240 $TR bench.py --gpus 2 --config $cfg $B > gpurun_out/e12_b2.json 2> gpurun_out/e12_b2.err; summ gpurun_out/e12_b2.json "n2 $cfg $kv"
  done
done
TRACE_GRAPH=1 timeout 200 $TR tools/trace_step.py dsv3_decode warp tma > gpurun_out/e12_trace2.log 2>&1; grep -A21 "rank 0\]" gpurun_out/e12_trace2.log | grep -E "layout.last|dispatch|combine"
