# round 2 (session 3), call 18 (4 GPUs): full GPU suite on 4 GPUs; EP=2/4 bench lines (default owner-reduce rule) +
# forced reduce at EP=4; driver-like lines at N=2 and N=4 for profiles/
set -x
export FUSCO_BENCH_WATCHDOG_S=150
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/e18_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/e18_pytest.log
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
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29700+N))"
  for cfg in mixtral qwen3 dsv3 dsv3_zipf dsv3_decode; do
    timeout 240 $TR bench.py --gpus $N --config $cfg $B > gpurun_out/e18_b${N}_$cfg.json 2> gpurun_out/e18_b${N}_$cfg.err; summ gpurun_out/e18_b${N}_$cfg.json "n$N $cfg"
  done
  FUSCO_BALANCE=0 timeout 240 $TR bench.py --gpus $N --config dsv3_zipf $B > gpurun_out/e18_b${N}_dsv3_zipf_bal0.json 2> gpurun_out/e18_bal0.err; summ gpurun_out/e18_b${N}_dsv3_zipf_bal0.json "n$N dsv3_zipf balance=0"
  FUSCO_OWNER_REDUCE=0 timeout 240 $TR bench.py --gpus $N --config dsv3_zipf $B > gpurun_out/e18_b${N}_dsv3_zipf_or0.json 2> gpurun_out/e18_or0.err; summ gpurun_out/e18_b${N}_dsv3_zipf_or0.json "n$N dsv3_zipf owner_reduce=0"
  FUSCO_OWNER_REDUCE=1 timeout 240 $TR bench.py --gpus $N --config dsv3_zipf $B > gpurun_out/e18_b${N}_dsv3_zipf_or1.json 2> gpurun_out/e18_or1.err; summ gpurun_out/e18_b${N}_dsv3_zipf_or1.json "n$N dsv3_zipf owner_reduce=1"
  FUSCO_OWNER_REDUCE=1 timeout 240 $TR bench.py --gpus $N --config dsv3 $B > gpurun_out/e18_b${N}_dsv3_or1.json 2> gpurun_out/e18_or1.err; summ gpurun_out/e18_b${N}_dsv3_or1.json "n$N dsv3 owner_reduce=1"
  timeout 600 $TR bench.py --gpus $N > gpurun_out/e18_bench_n$N.json 2> gpurun_out/e18_bench_n$N.err; echo "bench$N rc=$?"
  timeout 600 $TR bench.py --gpus $N --impl reference --steps 3 --warmup 1 > gpurun_out/e18_ref_n$N.json 2> gpurun_out/e18_ref_n$N.err; echo "ref$N rc=$?"
done
