# round 2 (re-entry), call 1 (2 GPUs): verify HEAD: gpu tests, smoke, N=1 bench + reference arm, N=2 bench, ncu of the N=1 line
set -x
nvidia-smi -L
timeout 1800 python -m pytest tests -m gpu -q -rs --durations=30 > gpurun_out/d1_pytest.log 2>&1; echo pytest_rc=$?
tail -45 gpurun_out/d1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/d1_smoke.log 2>&1; echo smoke_rc=$?
timeout 600 python bench.py > gpurun_out/d1_bench.json 2> gpurun_out/d1_bench.err; echo bench_rc=$?
cat gpurun_out/d1_bench.json; tail -5 gpurun_out/d1_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/d1_ref.json 2> gpurun_out/d1_ref.err; echo ref_rc=$?
cat gpurun_out/d1_ref.json
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29516"
timeout 600 $TR bench.py --gpus 2 > gpurun_out/d1_bench_n2.json 2> gpurun_out/d1_bench_n2.err; echo bench2_rc=$?
cat gpurun_out/d1_bench_n2.json; tail -5 gpurun_out/d1_bench_n2.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/d1_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --soak-s 0 > gpurun_out/d1_ncu1.log 2>&1; echo ncu1_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dispatch|combine|layout" -s 9 -c 3 -o gpurun_out/d1_dsv3z_full python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --soak-s 0 --eager > gpurun_out/d1_ncu2.log 2>&1; echo ncu2_rc=$?
ls -la gpurun_out
