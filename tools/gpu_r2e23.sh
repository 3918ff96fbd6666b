# round 2 (session 3), call 23 (4 GPUs): static fan-out / combine work at small batches: parity + decode benches
set -x
export FUSCO_BENCH_WATCHDOG_S=150
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multiproc.py -q -x > gpurun_out/e23_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/e23_pytest.log
summ() { python - "$1" "$2" <<'PY'
import json,sys
f=sys.argv[1]
try:
    d=json.loads([l for l in open(f) if l.startswith('{"metric"')][-1])
    print(sys.argv[2], round(d['latency_us'],1), {k:round(v,1) for k,v in d['kernel_us'].items()}, round(d['roofline_step_frac'],3))
except Exception as e: print(sys.argv[2], 'ERR', e)
PY
}
B="--steps 50 --warmup 5 --no-e2e --no-cpu-baseline"
for N in 2 4; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29750+N))"
  for rep in 1 2; do
    timeout 240 $TR bench.py --gpus $N --config dsv3_decode $B > gpurun_out/e23_b.json 2> gpurun_out/e23_b.err; summ gpurun_out/e23_b.json "n$N dsv3_decode"
  done
  TRACE_GRAPH=1 timeout 200 $TR tools/trace_step.py dsv3_decode warp tma > gpurun_out/e23_trace$N.log 2>&1; grep -A21 "rank 0\]" gpurun_out/e23_trace$N.log | grep -E "layout.last|dispatch|combine"
done
