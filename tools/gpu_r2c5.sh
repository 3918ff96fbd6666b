# round 2, call 5 (2 GPUs): per-kernel NVLink bytes by ncu (phased single-process run on 2 GPUs);
# cost of the per-unit release ordering of the block counts (FUSCO_DBG_BLK=1 = unordered, timing only)
set -x
export FUSCO_BENCH_WATCHDOG_S=150
M=gpu__time_duration.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum
for cfg in mixtral dsv3 qwen3; do
  timeout 300 python tools/ncu_nvlink.py --config $cfg --gpus 2 --iters 2 > gpurun_out/r2c5_nvl_plain_$cfg.log 2>&1 && \
  timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2c5_nvl_$cfg.csv python tools/ncu_nvlink.py --config $cfg --gpus 2 --iters 2 > gpurun_out/r2c5_nvl_ncu_$cfg.log 2>&1
  echo "nvl $cfg rc=$?"; tail -2 gpurun_out/r2c5_nvl_plain_$cfg.log
  python tools/ncu_nvlink.py --config $cfg --gpus 2 --summarize gpurun_out/r2c5_nvl_$cfg.csv > gpurun_out/r2c5_nvl_$cfg.json 2>&1; head -c 3000 gpurun_out/r2c5_nvl_$cfg.json
done
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514"
for cfg in mixtral dsv3; do
  FUSCO_DBG_BLK=1 TRACE_GRAPH=1 timeout 200 $TR tools/trace_step.py $cfg warp tma > gpurun_out/r2c5_trace_dbg_$cfg.log 2>&1; echo "trace $cfg rc=$?"
  grep -E "rank|dispatch|combine.ready" gpurun_out/r2c5_trace_dbg_$cfg.log | head -20
  FUSCO_DBG_BLK=1 timeout 200 $TR bench.py --gpus 2 --config $cfg --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2c5_dbg_$cfg.json 2>&1; echo "dbg $cfg rc=$?"
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2c5_dbg_*.json')):
    try:
        lines=[l for l in open(f) if l.startswith('{"metric"')]
        d=json.loads(lines[-1])
        print(f.split('/')[-1], round(d['latency_us'],1), {k:round(v,1) for k,v in d['kernel_us'].items()}, round(d['roofline_step_frac'],3))
    except Exception as e:
        print(f, 'ERR', e)
PY
