import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"
REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 CUDA devices")


def golden_names():
    return sorted(p.stem for p in GOLDEN.glob("*.npz"))


def load_golden(name):
    d = dict(np.load(GOLDEN / f"{name}.npz"))
    d["expert"] = str(d["expert"])
    for k in ("num_nodes", "gpus_per_node", "num_experts", "topk", "token_bytes", "payload_seed"):
        d[k] = int(d[k])
    return d


def split_rows(flat, rows, tb):
    """Concatenated per-rank byte buffers -> list of [rows, tb] arrays."""
    out, pos = [], 0
    for n in rows:
        out.append(flat[pos : pos + n * tb].reshape(n, tb))
        pos += n * tb
    return out


@pytest.fixture(scope="session")
def reference():
    """The live reference package, when this container has it (never on the GPU box)."""
    if not REFERENCE_SRC.exists():
        pytest.skip("reference not present")
    sys.path.insert(0, str(REFERENCE_SRC))
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    import shuffleforge

    return shuffleforge
