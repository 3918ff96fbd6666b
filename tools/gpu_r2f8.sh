# round 2 (session 3): full GPU suite on 2 GPUs with the final owner pass + the N=2 default line
set -x
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/f8_pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/f8_pytest.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29802"
timeout 600 $TR bench.py --gpus 2 > gpurun_out/f8_bench_n2.json 2> gpurun_out/f8_bench_n2.err; echo "bench2 rc=$?"
