# round 2 (session 3): ncu NVLink counters at EP=4 for DeepSeek-V3 / Zipf with the final default (owner
# pre-reduction on at P<=4 for 14 KB rows)
set -x
M=gpu__time_duration.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum
for cfg in dsv3 dsv3_zipf; do
  timeout 300 python tools/ncu_nvlink.py --config $cfg --gpus 4 --iters 2 > gpurun_out/f5_plain.log 2>&1 && \
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/f5_${cfg}_ep4.csv python tools/ncu_nvlink.py --config $cfg --gpus 4 --iters 2 > gpurun_out/f5_ncu_${cfg}.log 2>&1
  echo "$cfg rc=$?"
  python tools/ncu_nvlink.py --config $cfg --gpus 4 --summarize gpurun_out/f5_${cfg}_ep4.csv > gpurun_out/r2_nvl_counters_${cfg}_ep4.json 2>&1
done
