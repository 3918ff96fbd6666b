# round 2 (session 3), call 7 (4 GPUs): new pusher at EP=4: gpu tests on 4 GPUs, EP=4/EP=2 bench lines, balancer on/off,
# decode knobs, traces, HBM write ceiling
set -x
export FUSCO_BENCH_WATCHDOG_S=150
nvidia-smi -L
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/e7_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/e7_pytest.log
timeout 120 python tools/hbm_probe.py > gpurun_out/e7_hbm.json 2>&1; cat gpurun_out/e7_hbm.json
summ() { python - "$1" "$2" <<'PY'
import json,sys
f=sys.argv[1]
try:
    d=json.loads([l for l in open(f) if l.startswith('{"metric"')][-1])
    print(sys.argv[2], round(d['latency_us'],1), {k:round(v,1) for k,v in d['kernel_us'].items()}, round(d['roofline_step_frac'],3), d.get('nvlink_gbps_per_gpu'))
except Exception as e: print(sys.argv[2], 'ERR', e)
PY
}
B="--steps 30 --warmup 5 --no-e2e --no-cpu-baseline"
for N in 4 2; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29630+N))"
  for cfg in mixtral qwen3 dsv3 dsv3_zipf dsv3_decode; do
    timeout 240 $TR bench.py --gpus $N --config $cfg $B > gpurun_out/e7_b${N}_$cfg.json 2> gpurun_out/e7_b${N}_$cfg.err; summ gpurun_out/e7_b${N}_$cfg.json "n$N $cfg"
  done
  FUSCO_BALANCE=0 timeout 240 $TR bench.py --gpus $N --config dsv3_zipf $B > gpurun_out/e7_b${N}_dsv3_zipf_bal0.json 2> gpurun_out/e7_bal0.err; summ gpurun_out/e7_b${N}_dsv3_zipf_bal0.json "n$N dsv3_zipf balance=0"
  for kv in FUSCO_FAN_SPLIT=0 FUSCO_COMB_STAGE=8192 FUSCO_COMB_STAGE=12288 "FUSCO_COMB_STAGE=12288 FUSCO_TMA_CTAS=4"; do
    env $kv timeout 240 $TR bench.py --gpus $N --config dsv3_decode $B > gpurun_out/e7_dec.json 2> gpurun_out/e7_dec.err; summ gpurun_out/e7_dec.json "n$N dsv3_decode $kv"
  done
  for cfg in dsv3_decode dsv3_zipf; do
    TRACE_GRAPH=1 timeout 200 $TR tools/trace_step.py $cfg warp tma > gpurun_out/e7_trace${N}_$cfg.log 2>&1; echo "trace$N $cfg rc=$?"
  done
done
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29640"
timeout 600 $TR bench.py --gpus 4 > gpurun_out/e7_bench_n4.json 2> gpurun_out/e7_bench_n4.err; echo bench4_rc=$?; tail -1 gpurun_out/e7_bench_n4.json
