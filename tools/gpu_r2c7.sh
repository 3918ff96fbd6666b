# round 2, call 7 (2 GPUs): push rate of the TMA dispatch engine across GPUs (phased, ncu counters)
set -x
M=gpu__time_duration.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum
export FUSCO_DISPATCH=tma
for cfg in mixtral dsv3; do
  timeout 300 python tools/ncu_nvlink.py --config $cfg --gpus 2 --iters 2 > gpurun_out/r2c7_nvl_plain_$cfg.log 2>&1 && \
  timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2c7_nvl_tma_$cfg.csv python tools/ncu_nvlink.py --config $cfg --gpus 2 --iters 2 > gpurun_out/r2c7_nvl_ncu_$cfg.log 2>&1
  echo "nvl $cfg rc=$?"
  python tools/ncu_nvlink.py --config $cfg --gpus 2 --summarize gpurun_out/r2c7_nvl_tma_$cfg.csv > gpurun_out/r2c7_nvl_tma_$cfg.json 2>&1
done
for tc in 1 2 4; do
  FUSCO_TMA_CTAS=$tc timeout 300 python tools/ncu_nvlink.py --config dsv3 --gpus 2 --iters 2 > /dev/null 2>&1 && \
  FUSCO_TMA_CTAS=$tc timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2c7_nvl_tma${tc}_dsv3.csv python tools/ncu_nvlink.py --config dsv3 --gpus 2 --iters 2 > /dev/null 2>&1
  python tools/ncu_nvlink.py --config dsv3 --gpus 2 --summarize gpurun_out/r2c7_nvl_tma${tc}_dsv3.csv > gpurun_out/r2c7_nvl_tma${tc}_dsv3.json 2>&1
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2c7_nvl_tma*.json')):
    try:
        d=json.load(open(f))
        for k in d['kernels']:
            if k['kernel']=='fs_dispatch' and k['phase']=='local':
                print(f.split('/')[-1], k['gpu'], round(k['us'],1), round(k['nvl_tx_bytes']/1e6,2), round(k.get('nvl_tx_gbps',0)))
    except Exception as e:
        print(f, 'ERR', e)
PY
