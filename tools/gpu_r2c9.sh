# round 2, call 9 (2 GPUs): is the push limited by the dynamic claims? (static striding, phased, ncu); HBM mix ceilings
set -x
timeout 120 python tools/hbm_probe.py > gpurun_out/r2c9_hbm.json 2>&1; cat gpurun_out/r2c9_hbm.json
M=gpu__time_duration.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum
run() { tag=$1; cfg=$2; shift 2
  env "$@" timeout 300 python tools/ncu_nvlink.py --config $cfg --gpus 2 --iters 2 > /dev/null 2>&1 && \
  env "$@" timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2c9_${tag}_$cfg.csv python tools/ncu_nvlink.py --config $cfg --gpus 2 --iters 2 > /dev/null 2>&1
  echo "$tag $cfg rc=$?"
  python tools/ncu_nvlink.py --config $cfg --gpus 2 --summarize gpurun_out/r2c9_${tag}_$cfg.csv > gpurun_out/r2c9_${tag}_$cfg.json 2>&1
}
run static mixtral FUSCO_BALANCE=0
run static dsv3 FUSCO_BALANCE=0
run token mixtral FUSCO_CLAIM=token
run occ1 mixtral FUSCO_DISP_CTAS=1
run occ2 mixtral FUSCO_DISP_CTAS=2
run nodedup mixtral FUSCO_NODEDUP=1
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2c9_*_*.json')):
    try:
        d=json.load(open(f))
        for k in d['kernels']:
            if k['kernel']=='fs_dispatch':
                print(f.split('/')[-1], k['phase'], k['gpu'], round(k['us'],1), round(k['nvl_tx_bytes']/1e6,2), round(k.get('nvl_tx_gbps',0)), round(k['dram_bytes']/1e6,1))
    except Exception as e:
        print(f, 'ERR', e)
PY
