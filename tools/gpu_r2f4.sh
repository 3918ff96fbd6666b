# round 2 (session 3): the reference-style benchmark matrix on one B200 with the current kernels
# (balancer_off = the device knob fs_set_balance(h, 0), planner_off = no per-rank dedup)
set -x
timeout 1200 python -m paper_2512_22036_b200.matrix --preset box8 --repeats 2 --format json --out gpurun_out/r2_matrix_box8.json > gpurun_out/f4_matrix.log 2>&1; echo matrix_rc=$?
timeout 300 python -m paper_2512_22036_b200.matrix --preset box8 --repeats 1 --format md --out gpurun_out/r2_matrix_box8_quick.md > gpurun_out/f4_matrix_md.log 2>&1; echo md_rc=$?
tail -3 gpurun_out/f4_matrix.log
