# round 2, call 3 (2 GPUs): NVLink counter sources; dispatch claim granularity / grid sweep
set -x
export FUSCO_BENCH_WATCHDOG_S=150
timeout 120 python tools/nvlink_probe.py > gpurun_out/r2c3_nvprobe.json 2>&1; cat gpurun_out/r2c3_nvprobe.json
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x > gpurun_out/r2c3_mp_unit.log 2>&1; echo mp_unit_rc=$?; tail -3 gpurun_out/r2c3_mp_unit.log
FUSCO_CLAIM=token FUSCO_DISP_CTAS=1 timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x > gpurun_out/r2c3_mp_token.log 2>&1; echo mp_token_rc=$?; tail -3 gpurun_out/r2c3_mp_token.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512"
run() {  # tag env...
  tag=$1; shift
  for cfg in mixtral dsv3 dsv3_zipf qwen3 dsv3_decode; do
    env "$@" timeout 200 $TR bench.py --gpus 2 --config $cfg --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2c3_${tag}_$cfg.json 2>&1; echo "$tag $cfg rc=$?"
  done
}
run A FUSCO_CLAIM=unit
run B FUSCO_CLAIM=token
run C FUSCO_CLAIM=unit FUSCO_DISP_CTAS=1
run D FUSCO_CLAIM=token FUSCO_DISP_CTAS=1
run E FUSCO_CLAIM=token FUSCO_DISP_CTAS=2
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2c3_*_*.json')):
    try:
        lines=[l for l in open(f) if l.startswith('{"metric"')]
        d=json.loads(lines[-1])
        nv=d.get('nvlink_counters') or {}
        print(f.split('/')[-1], round(d['latency_us'],1), {k:round(v,1) for k,v in d['kernel_us'].items()}, round(d['roofline_step_frac'],3), nv.get('measured_over_algorithmic'), nv.get('unavailable'))
    except Exception as e:
        print(f, 'ERR', e)
PY
