# round 2 (session 3), call 13 (1 GPU): HBM ceilings of the P=1 dispatch's write pattern
set -x
timeout 200 python tools/hbm_probe.py > gpurun_out/e13_hbm.json 2>&1; cat gpurun_out/e13_hbm.json
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "push_rounds" 2>&1 | tail -2
