#!/bin/bash
# What the round-end driver runs, on all GPUs of the box: tests, smoke, N=1 bench + reference arm,
# then every N in 2..NGPU (powers of two) through torchrun, both arms.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/dl_pytest.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/dl_pytest.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/dl_smoke.log 2>&1; echo "smoke rc=$?"
for N in 1 2 4 8; do
  [ $N -gt $NG ] && break
  if [ $N -eq 1 ]; then
    timeout 600 python bench.py --impl reference > gpurun_out/dl_ref_n1.log 2>&1; echo "ref n=1 rc=$?"
    timeout 600 python bench.py > gpurun_out/dl_bench_n1.log 2>&1; echo "bench n=1 rc=$?"
  else
    RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29700 + N))"
    timeout 600 $RUN bench.py --impl reference --gpus $N > gpurun_out/dl_ref_n$N.log 2>&1; echo "ref n=$N rc=$?"
    timeout 600 $RUN bench.py --gpus $N > gpurun_out/dl_bench_n$N.log 2>&1; echo "bench n=$N rc=$?"
  fi
  tail -1 gpurun_out/dl_bench_n$N.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('  value',round(d['value'],1),d['unit'],'ms',round(d['ms_per_step']*1e3,1),'us','e2e',round(d['e2e']['value'],1),'frac',round(d['roofline']['frac'],3))" 2>&1 | tail -1
  tail -1 gpurun_out/dl_ref_n$N.log | cut -c1-160
done
