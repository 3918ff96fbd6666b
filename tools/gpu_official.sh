#!/bin/bash
# Driver-equivalent runs on 1 GPU + ncu evidence for profiles/.  Usage: bash tools/gpu_official.sh <tag>
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu_${TAG}.log
timeout 600 python bench.py > gpurun_out/bench_default_${TAG}.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_default_${TAG}.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_${TAG}.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref_${TAG}.log
CMD="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --soak-s 0 --eager"
$CMD > gpurun_out/plain_ncu_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"layout_kernel|dispatch|combine" --csv --log-file gpurun_out/launches_default_${TAG}.csv $CMD \
    > gpurun_out/ncu_launch_default_${TAG}.log 2>&1
echo "launch-list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"layout_kernel|dispatch|combine" -s 30 -c 3 \
    -o gpurun_out/prof_default_${TAG} -f $CMD > gpurun_out/ncu_full_default_${TAG}.log 2>&1
echo "ncu-full rc=$?"
