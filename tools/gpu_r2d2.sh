# round 2 (re-entry), call 2 (4 GPUs): EP=4/EP=2 bench lines, balancer on/off, per-phase timelines,
# ncu NVLink counters at 4 GPUs, HBM access-mix ceilings
set -x
export FUSCO_BENCH_WATCHDOG_S=150
timeout 120 python tools/hbm_probe.py > gpurun_out/d2_hbm.json 2>&1; cat gpurun_out/d2_hbm.json
B="--steps 30 --warmup 5 --no-e2e --no-cpu-baseline"
for N in 4 2; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600+N))"
  CF="mixtral qwen3 dsv3 dsv3_decode dsv3_zipf"; [ $N -eq 2 ] && CF="dsv3_decode dsv3 mixtral"
  for cfg in $CF; do
    timeout 240 $TR bench.py --gpus $N --config $cfg $B > gpurun_out/d2_b${N}_$cfg.json 2> gpurun_out/d2_b${N}_$cfg.err; echo "b$N $cfg rc=$?"
  done
  FUSCO_BALANCE=0 timeout 240 $TR bench.py --gpus $N --config dsv3_zipf $B > gpurun_out/d2_b${N}_dsv3_zipf_bal0.json 2> gpurun_out/d2_b${N}_bal0.err; echo "bal0 $N rc=$?"
  for cfg in dsv3_decode dsv3_zipf dsv3; do
    TRACE_GRAPH=1 timeout 200 $TR tools/trace_step.py $cfg warp tma > gpurun_out/d2_trace${N}_$cfg.log 2>&1; echo "trace$N $cfg rc=$?"
  done
done
M=gpu__time_duration.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum
for cfg in mixtral dsv3 qwen3 dsv3_zipf; do
  timeout 300 python tools/ncu_nvlink.py --config $cfg --gpus 4 --iters 2 > gpurun_out/d2_nvl_plain_$cfg.log 2>&1 && \
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/d2_nvl4_$cfg.csv python tools/ncu_nvlink.py --config $cfg --gpus 4 --iters 2 > gpurun_out/d2_nvl_ncu_$cfg.log 2>&1
  echo "nvl $cfg rc=$?"
  python tools/ncu_nvlink.py --config $cfg --gpus 4 --summarize gpurun_out/d2_nvl4_$cfg.csv > gpurun_out/r2_nvl_counters_${cfg}_ep4.json 2>&1
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/d2_b*.json')):
    try:
        lines=[l for l in open(f) if l.startswith('{"metric"')]
        d=json.loads(lines[-1])
        print(f.split('/')[-1], round(d['latency_us'],1), {k:round(v,1) for k,v in d['kernel_us'].items()}, round(d['roofline_step_frac'],3))
    except Exception as e:
        print(f, 'ERR', e)
PY
