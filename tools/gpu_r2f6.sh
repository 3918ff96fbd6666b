# round 2 (session 3): final bench.py check at N=2 / N=4 (reporting change: counter bytes in the roofline)
set -x
for N in 2 4; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29780+N))"
  timeout 600 $TR bench.py --gpus $N > gpurun_out/f6_bench_n$N.json 2> gpurun_out/f6_bench_n$N.err; echo "bench$N rc=$?"
  python -c "import json;d=json.loads([l for l in open('gpurun_out/f6_bench_n$N.json') if l.startswith('{\"metric\"')][-1]);print($N, round(d['latency_us'],1), d['roofline'])"
done
