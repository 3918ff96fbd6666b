# round 2 (session 3), call 9 (1 GPU): sliced last round in the TMA dispatch: parity, A/B, ncu full of the dispatch
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_acceptance.py -q -x > gpurun_out/e9_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/e9_pytest.log
summ() { python - "$1" "$2" <<'PY'
import json,sys
f=sys.argv[1]
try:
    d=json.loads([l for l in open(f) if l.startswith('{"metric"')][-1])
    print(sys.argv[2], round(d['latency_us'],1), {k:round(v,1) for k,v in d['kernel_us'].items()}, round(d['roofline_step_frac'],3))
except Exception as e: print(sys.argv[2], 'ERR', e)
PY
}
B1="--steps 100 --warmup 5 --no-e2e --no-cpu-baseline"
for rep in 1 2; do
for cfg in dsv3_zipf mixtral qwen3; do
  for kv in BASE=1 FUSCO_TMA_TAIL=0; do
    env $kv timeout 200 python bench.py --config $cfg $B1 > gpurun_out/e9.json 2>gpurun_out/e9.err; summ gpurun_out/e9.json "n1 $cfg $kv"
  done
done
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dispatch_tma|combine_kernel" -s 4 -c 2 -o gpurun_out/e9_full python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --soak-s 0 --eager > gpurun_out/e9_ncu.log 2>&1; echo ncu_rc=$?
ls -la gpurun_out/ | grep e9_full
