# round 2 (session 3), call 4 (2 GPUs): bisect the P>1 push regression (r1 -> a3cb7cd -> b6a7e98 -> HEAD), P=1 TMA dispatch sweep
set -x
ROOT=$(pwd)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29519"
B="--steps 30 --warmup 5 --no-e2e --no-cpu-baseline"
summ() { python - "$1" "$2" <<'PY'
import json,sys
f=sys.argv[1]
try:
    d=json.loads([l for l in open(f) if l.startswith('{"metric"')][-1])
    print(sys.argv[2], round(d['latency_us'],1), {k:round(v,1) for k,v in d['kernel_us'].items()}, round(d['roofline_step_frac'],3))
except Exception as e: print(sys.argv[2], 'ERR', e)
PY
}
for cfg in mixtral dsv3; do
  for t in r1 a3cb7cd b6a7e98; do
    (cd _ab/$t && timeout 240 $TR bench.py --gpus 2 --config $cfg $B > $ROOT/gpurun_out/e4.json 2> $ROOT/gpurun_out/e4_$t.err); summ gpurun_out/e4.json "n2 $cfg $t"
  done
  timeout 240 $TR bench.py --gpus 2 --config $cfg $B > gpurun_out/e4.json 2> gpurun_out/e4_hd.err; summ gpurun_out/e4.json "n2 $cfg HEAD"
done
B1="--steps 50 --warmup 5 --no-e2e --no-cpu-baseline"
for cfg in dsv3_zipf mixtral qwen3; do
  for kv in "FUSCO_TMA_SLICES=1" "FUSCO_TMA_LAG=4" "FUSCO_TMA_LAG=4 FUSCO_TMA_SLICES=2" "FUSCO_TMA_CTAS=4" "FUSCO_TMA_CTAS=2" "FUSCO_TMA_CTAS=4 FUSCO_TMA_LAG=4" "FUSCO_TMA_CTAS=6 FUSCO_TMA_LAG=4 FUSCO_TMA_SLICES=2"; do
    env $kv timeout 200 python bench.py --config $cfg $B1 > gpurun_out/e4.json 2>gpurun_out/e4_n1.err; summ gpurun_out/e4.json "n1 $cfg $kv"
  done
done
