# round 2, call 4 (2 GPUs): timelines of the block-signalled dispatch; the DSV3-Zipf hang hunt
set -x
export FUSCO_BENCH_WATCHDOG_S=150
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513"
for cfg in mixtral dsv3 dsv3_decode dsv3_zipf; do
  TRACE_GRAPH=1 timeout 200 $TR tools/trace_step.py $cfg warp tma > gpurun_out/r2c4_trace_$cfg.log 2>&1; echo "trace $cfg rc=$?"
  grep -v "^\*\|OMP\|NCCL" gpurun_out/r2c4_trace_$cfg.log | head -60
done
for it in 1 2 3 4 5; do
  timeout 200 $TR bench.py --gpus 2 --config dsv3_zipf --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2c4_zipf_$it.json 2>&1; echo "zipf $it rc=$?"
  grep -E "FuscoError|timed out|Timeout|Error" gpurun_out/r2c4_zipf_$it.json | head -5
done
FUSCO_PUSH_WARPS=7 timeout 200 $TR bench.py --gpus 2 --config mixtral --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2c4_pw7_mixtral.json 2>&1; echo "pw7 rc=$?"
FUSCO_PUSH_WARPS=7 timeout 200 $TR bench.py --gpus 2 --config dsv3 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2c4_pw7_dsv3.json 2>&1; echo "pw7 rc=$?"
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2c4_*.json')):
    try:
        lines=[l for l in open(f) if l.startswith('{"metric"')]
        d=json.loads(lines[-1])
        print(f.split('/')[-1], round(d['latency_us'],1), {k:round(v,1) for k,v in d['kernel_us'].items()}, round(d['roofline_step_frac'],3))
    except Exception as e:
        print(f, 'ERR', e)
PY
