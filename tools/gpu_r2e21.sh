# round 2 (session 3), call 21 (1 GPU): P=1 combine engine A/B (TMA vs warp) and stage size on the headline config
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
B1="--steps 100 --warmup 5 --no-e2e --no-cpu-baseline"
for cfg in dsv3_zipf qwen3 mixtral; do
  for kv in BASE=1 FUSCO_COMBINE=tma "FUSCO_COMBINE=tma FUSCO_COMB_STAGE=49152" "FUSCO_COMBINE=tma FUSCO_COMB_STAGE=12288" "FUSCO_COMBINE=tma FUSCO_TMA_CTAS=2"; do
    env $kv timeout 200 python bench.py --config $cfg $B1 > gpurun_out/e21.json 2>gpurun_out/e21.err; summ gpurun_out/e21.json "n1 $cfg $kv"
  done
done
