# round 2 (session 3), call 8 (1 GPU): P=1 dispatch engines/shapes on the headline config, ncu full of the TMA dispatch
set -x
summ() { python - "$1" "$2" <<'PY'
import json,sys
f=sys.argv[1]
try:
    d=json.loads([l for l in open(f) if l.startswith('{"metric"')][-1])
    print(sys.argv[2], round(d['latency_us'],1), {k:round(v,1) for k,v in d['kernel_us'].items()}, round(d['roofline_step_frac'],3))
except Exception as e: print(sys.argv[2], 'ERR', e)
PY
}
B1="--steps 50 --warmup 5 --no-e2e --no-cpu-baseline"
for cfg in dsv3_zipf mixtral; do
  for kv in BASE=1 FUSCO_DISPATCH=warp "FUSCO_TMA_CTAS=2 FUSCO_TMA_LAG=4" "FUSCO_TMA_CTAS=1 FUSCO_TMA_LAG=4" "FUSCO_TMA_CTAS=8" "FUSCO_PDL=0"; do
    env $kv timeout 200 python bench.py --config $cfg $B1 > gpurun_out/e8.json 2>gpurun_out/e8.err; summ gpurun_out/e8.json "n1 $cfg $kv"
  done
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dispatch_tma" -s 6 -c 2 -o gpurun_out/e8_disp_full python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --soak-s 0 --eager > gpurun_out/e8_ncu.log 2>&1; echo ncu_rc=$?
ls -la gpurun_out/e8_disp_full*
