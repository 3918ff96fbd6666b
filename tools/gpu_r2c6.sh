# round 2, call 6 (2 GPUs): dispatch at 64 registers (4 CTAs/SM); probe reference; counters; bench
set -x
export FUSCO_BENCH_WATCHDOG_S=150
M=gpu__time_duration.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29515"
timeout 300 $TR tools/p2p_probe.py > gpurun_out/r2c6_probe.log 2>&1; echo probe rc=$?; grep world gpurun_out/r2c6_probe.log
for cfg in mixtral dsv3; do
  timeout 300 python tools/ncu_nvlink.py --config $cfg --gpus 2 --iters 2 > gpurun_out/r2c6_nvl_plain_$cfg.log 2>&1 && \
  timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2c6_nvl_$cfg.csv python tools/ncu_nvlink.py --config $cfg --gpus 2 --iters 2 > gpurun_out/r2c6_nvl_ncu_$cfg.log 2>&1
  echo "nvl $cfg rc=$?"
  python tools/ncu_nvlink.py --config $cfg --gpus 2 --summarize gpurun_out/r2c6_nvl_$cfg.csv > gpurun_out/r2c6_nvl_$cfg.json 2>&1
done
for cfg in mixtral dsv3 qwen3 dsv3_decode dsv3_zipf; do
  timeout 200 $TR bench.py --gpus 2 --config $cfg --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2c6_b_$cfg.json 2>&1; echo "b $cfg rc=$?"
done
TRACE_GRAPH=1 timeout 200 $TR tools/trace_step.py mixtral warp tma > gpurun_out/r2c6_trace_mixtral.log 2>&1; echo "trace rc=$?"
grep -E "rank|dispatch|combine" gpurun_out/r2c6_trace_mixtral.log | head -24
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2c6_b_*.json')):
    try:
        lines=[l for l in open(f) if l.startswith('{"metric"')]
        d=json.loads(lines[-1])
        print(f.split('/')[-1], round(d['latency_us'],1), {k:round(v,1) for k,v in d['kernel_us'].items()}, round(d['roofline_step_frac'],3))
    except Exception as e:
        print(f, 'ERR', e)
for c in ['mixtral','dsv3']:
    try:
        d=json.load(open(f'gpurun_out/r2c6_nvl_{c}.json'))
        for k in d['kernels']:
            if k['kernel']!='fs_layout' and k['us']>10:
                print(c, k['kernel'], k['phase'], k['gpu'], round(k['us'],1), round(k['nvl_tx_bytes']/1e6,2), round(k['nvl_rx_bytes']/1e6,2), round(k.get('nvl_tx_gbps',0)), round(k.get('nvl_rx_gbps',0)))
    except Exception as e:
        print(c, 'ERR', e)
PY
