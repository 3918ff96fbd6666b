# round 2 (session 3), call 20 (4 GPUs): final default (owner pre-reduction at P<=4 for >= 8 KB rows): GPU suite,
# EP=4 bench lines, driver-like N=2 / N=4 lines
set -x
export FUSCO_BENCH_WATCHDOG_S=150
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/e20_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/e20_pytest.log
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
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29740"
for cfg in dsv3 dsv3_zipf qwen3 mixtral dsv3_decode; do
  timeout 240 $TR bench.py --gpus 4 --config $cfg $B > gpurun_out/e20_b4_$cfg.json 2> gpurun_out/e20_b4_$cfg.err; summ gpurun_out/e20_b4_$cfg.json "n4 $cfg"
done
timeout 600 $TR bench.py --gpus 4 > gpurun_out/e20_bench_n4.json 2> gpurun_out/e20_bench_n4.err; echo "bench4 rc=$?"
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29742"
timeout 600 $TR2 bench.py --gpus 2 > gpurun_out/e20_bench_n2.json 2> gpurun_out/e20_bench_n2.err; echo "bench2 rc=$?"
TRACE_GRAPH=1 timeout 200 $TR tools/trace_step.py dsv3_zipf warp tma > gpurun_out/e20_trace4_zipf.log 2>&1; echo trace_rc=$?
