# round 2 (session 3), final driver-equivalent sequence on 4 GPUs (tests, smoke, both arms at N=1,2,4), plus a
# decode A/B (per-CTA-round counting at EP=4)
set -x
export FUSCO_BENCH_WATCHDOG_S=200
bash tools/driver_like.sh
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29760"
for kv in FUSCO_PUSH_ROUNDS=1 BASE=1; do
  env $kv timeout 240 $TR bench.py --gpus 4 --config dsv3_decode --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/f2_dec.json 2>&1
  python -c "import json;d=json.loads([l for l in open('gpurun_out/f2_dec.json') if l.startswith('{\"metric\"')][-1]);print('n4 decode $kv',round(d['latency_us'],1),d['kernel_us'])"
done
