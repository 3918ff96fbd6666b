# round 2 (session 3): owner pass with one-round-trip records and both chunks' loads together: parity + EP=2/4
set -x
export FUSCO_BENCH_WATCHDOG_S=150
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "owner_reduce" > gpurun_out/f7_pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/f7_pytest.log
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x -k "256-1 or 300-1 or 7168" > gpurun_out/f7_pytest2.log 2>&1; echo pytest2_rc=$?; tail -2 gpurun_out/f7_pytest2.log
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
for N in 4 2; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29790+N))"
  for cfg in dsv3 dsv3_zipf; do
    timeout 240 $TR bench.py --gpus $N --config $cfg $B > gpurun_out/f7_b.json 2> gpurun_out/f7_b.err; summ gpurun_out/f7_b.json "n$N $cfg"
  done
done
