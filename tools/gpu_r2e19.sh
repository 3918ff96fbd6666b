# round 2 (session 3), call 19 (4 GPUs): ncu NVLink TX/RX counters per kernel for the current code at EP=2 (owner
# pre-reduction on by default there) and EP=4 (default off; dsv3_zipf also forced on)
set -x
export FUSCO_BENCH_WATCHDOG_S=150
summ() { python - "$1" "$2" <<'PY2'
import json,sys
f=sys.argv[1]
try:
    d=json.loads([l for l in open(f) if l.startswith('{"metric"')][-1])
    print(sys.argv[2], round(d['latency_us'],1), {k:round(v,1) for k,v in d['kernel_us'].items()}, round(d['roofline_step_frac'],3), d.get('owner_reduce'))
except Exception as e: print(sys.argv[2], 'ERR', e)
PY2
}
B="--steps 30 --warmup 5 --no-e2e --no-cpu-baseline"
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29720"
for cfg in qwen3 dsv3_decode; do
  for kv in FUSCO_OWNER_REDUCE=1 BASE=1; do
    env $kv timeout 240 $TR bench.py --gpus 4 --config $cfg $B > gpurun_out/e19_b.json 2> gpurun_out/e19_b.err; summ gpurun_out/e19_b.json "n4 $cfg $kv"
  done
done
M=gpu__time_duration.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum
run() { tag=$1; cfg=$2; G=$3; shift 3
  env "$@" timeout 300 python tools/ncu_nvlink.py --config $cfg --gpus $G --iters 2 > gpurun_out/e19_plain.log 2>&1 && \
  env "$@" timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/e19_${tag}.csv python tools/ncu_nvlink.py --config $cfg --gpus $G --iters 2 > gpurun_out/e19_ncu_${tag}.log 2>&1
  echo "$tag rc=$?"
  python tools/ncu_nvlink.py --config $cfg --gpus $G --summarize gpurun_out/e19_${tag}.csv > gpurun_out/r2_nvl_counters_${tag}.json 2>&1
}
for cfg in dsv3 dsv3_zipf mixtral qwen3; do run ${cfg}_ep2 $cfg 2 X=1; done
for cfg in dsv3 dsv3_zipf mixtral qwen3; do run ${cfg}_ep4 $cfg 4 X=1; done
run dsv3_zipf_ep4_or1 dsv3_zipf 4 FUSCO_OWNER_REDUCE=1
python tools/nvl_table.py gpurun_out/r2_nvl_counters_*.json > gpurun_out/r2_nvlink_counters_table.md; cat gpurun_out/r2_nvlink_counters_table.md
