# round 2 (session 3), call 24 (4 GPUs): owner pass overlapped with the pulls (per-(source, block) partial flags,
# a third of the CTAs run the pass): parity + A/B at EP=2/4
set -x
export FUSCO_BENCH_WATCHDOG_S=150
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multiproc.py -q -x -k "owner_reduce or multi_gpu or bf16_parity or engine_parity" > gpurun_out/e24_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/e24_pytest.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "ep2 or zipf-ep4 or reduce" > gpurun_out/e24_pytest2.log 2>&1; echo pytest2_rc=$?; tail -3 gpurun_out/e24_pytest2.log
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
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29770+N))"
  for cfg in dsv3 dsv3_zipf qwen3; do
    for kv in BASE=1 FUSCO_REDUCE_CTAS=0 FUSCO_REDUCE_CTAS=74 "FUSCO_OWNER_REDUCE=1 X=1"; do
      env $kv timeout 240 $TR bench.py --gpus $N --config $cfg $B > gpurun_out/e24_b.json 2> gpurun_out/e24_b.err; summ gpurun_out/e24_b.json "n$N $cfg $kv"
    done
  done
done
