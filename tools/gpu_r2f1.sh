# round 2 (session 3), final-ish 1-GPU evidence: driver-equivalent tests/smoke/bench/reference arm + ncu launch list + full set
set -x
bash tools/gpu_official.sh r2f
tail -2 gpurun_out/bench_default_r2f.log | cut -c1-400
python tools/ncu_summary.py r2 dsv3_zipf 1 gpurun_out/launches_default_r2f.csv gpurun_out/prof_default_r2f.ncu-rep > gpurun_out/ncu_summary_r2f.log 2>&1; echo summary_rc=$?
ls -la profiles | tail -5
