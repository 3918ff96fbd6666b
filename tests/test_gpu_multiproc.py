"""Real multi-GPU path (one process per GPU, NVLink P2P through CUDA IPC),
checked against the oracle by every rank.  Runs with as many GPUs as the
box exposes (2, 4 or 8); skipped on a 1-GPU box."""

import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

ROOT = Path(__file__).resolve().parent.parent


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("experts,topk,hidden,dtype,engines,tokens,reduce", [
    (64, 8, 2048, "bf16", "auto:auto", 256, ""),
    (64, 8, 2048, "bf16", "auto:auto", 256, "1"),   # owner pre-reduction forced on at any world size
    (16, 4, 1024, "f32", "auto:auto", 300, "1"),    # ... with fp32 rows (groups of >= 2)
    (8, 2, 2048, "bf16", "auto:auto", 256, ""),
    (32, 4, 1030, "bf16", "auto:auto", 256, ""),   # 2060-byte rows: not a multiple of 16, the 4-byte movers
    (16, 4, 1024, "f32", "auto:auto", 256, ""),    # fp32 payload, f64-accumulate combine bit-exact
    (64, 8, 2048, "bf16", "tma:warp", 256, ""),    # the other data movers across GPUs
    (256, 8, 7168, "bf16", "auto:auto", 4096, ""),  # DeepSeek-V3 shape at the BASELINE batch
    (8, 2, 4096, "bf16", "auto:auto", 8192, ""),   # Mixtral shape at the BASELINE batch
])
def test_multi_gpu_parity(experts, topk, hidden, dtype, engines, tokens, reduce):
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(n, 8)
    if experts % world:
        pytest.skip("experts not divisible by world")
    d, c = engines.split(":")
    env = dict(os.environ, MP_E=str(experts), MP_K=str(topk), MP_H=str(hidden), MP_DT=dtype,
               MP_T=str(tokens), MP_ITERS="4" if tokens <= 1024 else "2", FUSCO_DISPATCH=d, FUSCO_COMBINE=c)
    if reduce:
        env["FUSCO_OWNER_REDUCE"] = reduce
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "tests" / "mp_worker.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert res.returncode == 0, res.stdout[-4000:] + res.stderr[-4000:]
    assert "failures=0" in res.stdout
