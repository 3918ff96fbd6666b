# round 2 (session 3), call 2 (2 GPUs): A/B round-1 tree vs HEAD at EP=2, and HEAD dispatch knobs
set -x
ROOT=$(pwd)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517"
B="--steps 30 --warmup 5 --no-e2e --no-cpu-baseline"
summ() { python - "$1" <<'PY'
import json,sys
f=sys.argv[1]
try:
    d=json.loads([l for l in open(f) if l.startswith('{"metric"')][-1])
    print(f.split('/')[-1], round(d['latency_us'],1), {k:round(v,1) for k,v in d['kernel_us'].items()}, round(d['roofline_step_frac'],3))
except Exception as e: print(f, 'ERR', e)
PY
}
for cfg in mixtral dsv3_decode qwen3 dsv3; do
  (cd _ab/r1 && timeout 240 $TR bench.py --gpus 2 --config $cfg $B > $ROOT/gpurun_out/e2_r1_$cfg.json 2> $ROOT/gpurun_out/e2_r1_$cfg.err); summ gpurun_out/e2_r1_$cfg.json
  timeout 240 $TR bench.py --gpus 2 --config $cfg $B > gpurun_out/e2_hd_$cfg.json 2> gpurun_out/e2_hd_$cfg.err; summ gpurun_out/e2_hd_$cfg.json
done
for kv in FUSCO_DBG_BLK=1 FUSCO_CLAIM=token FUSCO_PUSH_WARPS=6 FUSCO_PUSH_WARPS=4 FUSCO_BALANCE=0; do
  for cfg in mixtral dsv3_decode; do
    env $kv timeout 240 $TR bench.py --gpus 2 --config $cfg $B > gpurun_out/e2_${kv}_$cfg.json 2> gpurun_out/e2_${kv}_$cfg.err; summ gpurun_out/e2_${kv}_$cfg.json
  done
done
for cfg in mixtral dsv3_decode; do
  (cd _ab/r1 && TRACE_GRAPH=1 timeout 200 $TR tools/trace_step.py $cfg warp tma > $ROOT/gpurun_out/e2_r1_trace_$cfg.log 2>&1)
  TRACE_GRAPH=1 timeout 200 $TR tools/trace_step.py $cfg warp tma > gpurun_out/e2_hd_trace_$cfg.log 2>&1
done
