# round 2 (session 3), call 22 (2 GPUs): new owner-reduce parity tests (full size, ragged mixed decisions) + suite
set -x
timeout 1800 python -m pytest tests -m gpu -q -x -rs > gpurun_out/e22_pytest.log 2>&1; echo pytest_rc=$?; tail -8 gpurun_out/e22_pytest.log
