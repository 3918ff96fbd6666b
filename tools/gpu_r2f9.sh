# round 2 (session 3): the N=4 default line with the final owner pass
set -x
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29804"
timeout 400 $TR bench.py --gpus 4 > gpurun_out/f9_bench_n4.json 2> gpurun_out/f9_bench_n4.err; echo "bench4 rc=$?"
