# round 2, call 2 (2 GPUs): block-signalled dispatch — parity (emulated + real 2-process), NVLink counters, bench
set -x
nvidia-smi topo -m | head -5
timeout 120 python tools/nvlink_probe.py > gpurun_out/r2c2_nvprobe.json 2>&1; cat gpurun_out/r2c2_nvprobe.json
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/r2c2_pytest.log 2>&1; echo pytest_rc=$?
tail -25 gpurun_out/r2c2_pytest.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
for cfg in dsv3_zipf dsv3 mixtral qwen3 dsv3_decode; do
  timeout 300 $TR bench.py --gpus 2 --config $cfg --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2c2_b_$cfg.json 2> gpurun_out/r2c2_b_$cfg.err; echo "$cfg rc=$?"
  tail -c 1500 gpurun_out/r2c2_b_$cfg.json; tail -3 gpurun_out/r2c2_b_$cfg.err
done
for pw in 6 4; do
  for cfg in dsv3_zipf dsv3; do
    FUSCO_PUSH_WARPS=$pw timeout 300 $TR bench.py --gpus 2 --config $cfg --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2c2_pw${pw}_$cfg.json 2>&1; echo "pw=$pw $cfg rc=$?"
  done
done
FUSCO_BALANCE=0 timeout 300 $TR bench.py --gpus 2 --config dsv3_zipf --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2c2_bal0_dsv3_zipf.json 2>&1; echo "bal0 rc=$?"
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2c2_*.json')):
    try:
        lines=[l for l in open(f) if l.startswith('{"metric"')]
        d=json.loads(lines[-1])
        nv=d.get('nvlink_counters') or {}
        print(f, round(d['latency_us'],1), {k:round(v,1) for k,v in d['kernel_us'].items()}, round(d['roofline_step_frac'],3), nv.get('measured_over_algorithmic'))
    except Exception as e:
        print(f, 'ERR', e)
PY
