# round 2 (session 3), call 17 (4 GPUs): owner pre-reduction with column-split work: parity at 4 GPUs, EP=2/4 A/B
set -x
export FUSCO_BENCH_WATCHDOG_S=150
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multiproc.py -q -x > gpurun_out/e17_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/e17_pytest.log
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
for N in 2 4; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29690+N))"
  for cfg in dsv3_decode dsv3 dsv3_zipf qwen3; do
    for kv in BASE=1 FUSCO_OWNER_REDUCE=0; do
      env $kv timeout 240 $TR bench.py --gpus $N --config $cfg $B > gpurun_out/e17_b.json 2> gpurun_out/e17_b.err; summ gpurun_out/e17_b.json "n$N $cfg $kv"
    done
  done
done
