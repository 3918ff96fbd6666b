# round 2 (session 3), call 1 (2 GPUs): verify HEAD after re-entry: gpu tests, smoke, N=1/N=2 bench, balancer on/off at EP=2
set -x
nvidia-smi -L
timeout 1800 python -m pytest tests -m gpu -q -rs --durations=25 > gpurun_out/e1_pytest.log 2>&1; echo pytest_rc=$?
tail -40 gpurun_out/e1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e1_smoke.log 2>&1; echo smoke_rc=$?
timeout 600 python bench.py > gpurun_out/e1_bench.json 2> gpurun_out/e1_bench.err; echo bench_rc=$?
cat gpurun_out/e1_bench.json; tail -3 gpurun_out/e1_bench.err
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29516"
B="--steps 30 --warmup 5 --no-e2e --no-cpu-baseline"
for cfg in dsv3_zipf dsv3 mixtral qwen3 dsv3_decode; do
  timeout 240 $TR bench.py --gpus 2 --config $cfg $B > gpurun_out/e1_b2_$cfg.json 2> gpurun_out/e1_b2_$cfg.err; echo "b2 $cfg rc=$?"
done
FUSCO_BALANCE=0 timeout 240 $TR bench.py --gpus 2 --config dsv3_zipf $B > gpurun_out/e1_b2_dsv3_zipf_bal0.json 2> gpurun_out/e1_b2_bal0.err; echo "bal0 rc=$?"
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/e1_b*.json')):
    try:
        lines=[l for l in open(f) if l.startswith('{"metric"')]
        d=json.loads(lines[-1])
        print(f.split('/')[-1], round(d['latency_us'],1), {k:round(v,1) for k,v in d['kernel_us'].items()}, round(d['roofline_step_frac'],3))
    except Exception as e:
        print(f, 'ERR', e)
PY
