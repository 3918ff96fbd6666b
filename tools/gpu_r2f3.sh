# round 2 (session 3), final 1-GPU check of HEAD: GPU suite, smoke, default bench line
set -x
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/f3_pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/f3_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3_smoke.log 2>&1; echo smoke_rc=$?
timeout 600 python bench.py > gpurun_out/f3_bench.json 2> gpurun_out/f3_bench.err; echo bench_rc=$?
python -c "import json;d=json.loads(open('gpurun_out/f3_bench.json').read().splitlines()[-1]);print(d['latency_us'],d['roofline_step_frac'],d['roofline']['frac'],d['roofline'].get('pattern_ceiling',{}).get('frac'),d['e2e']['value'],d['clocks'])"
