# round 2 (session 3), call 11 (4 GPUs): small-batch static push with PDL-overlapped payload loads: tests + decode/large benches
set -x
export FUSCO_BENCH_WATCHDOG_S=150
timeout 1500 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x > gpurun_out/e11_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/e11_pytest.log
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
for N in 2 4; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29650+N))"
  for cfg in dsv3_decode mixtral dsv3; do
    timeout 240 $TR bench.py --gpus $N --config $cfg $B > gpurun_out/e11_b${N}_$cfg.json 2> gpurun_out/e11_b${N}_$cfg.err; summ gpurun_out/e11_b${N}_$cfg.json "n$N $cfg"
  done
  TRACE_GRAPH=1 timeout 200 $TR tools/trace_step.py dsv3_decode warp tma > gpurun_out/e11_trace${N}.log 2>&1; echo "trace$N rc=$?"
  grep -A21 "rank 0\]" gpurun_out/e11_trace${N}.log | grep -E "layout.last|dispatch|combine"
done
