set -x
nvidia-smi -L
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=25 > gpurun_out/r2c1_pytest.log 2>&1; echo pytest_rc=$?
tail -40 gpurun_out/r2c1_pytest.log
timeout 300 python __graft_entry__.py > gpurun_out/r2c1_smoke.log 2>&1; echo smoke_rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2c1_bench.json 2> gpurun_out/r2c1_bench.err; echo bench_rc=$?
cat gpurun_out/r2c1_bench.json; tail -5 gpurun_out/r2c1_bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2c1_ref.json 2> gpurun_out/r2c1_ref.err; echo ref_rc=$?
cat gpurun_out/r2c1_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2c1_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --soak-s 0 > gpurun_out/r2c1_ncu1.log 2>&1; echo ncu1_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dispatch -s 6 -c 1 -o gpurun_out/r2c1_dsv3z_dispatch python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --soak-s 0 --eager > gpurun_out/r2c1_ncu2.log 2>&1; echo ncu2_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:combine -s 6 -c 1 -o gpurun_out/r2c1_dsv3z_combine python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --soak-s 0 --eager > gpurun_out/r2c1_ncu3.log 2>&1; echo ncu3_rc=$?
ls -la gpurun_out
