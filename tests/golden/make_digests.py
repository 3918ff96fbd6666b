"""Reference digests at full BASELINE sizes (the arrays are too large to commit).

Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_digests.py [case ...]

For each case the reference ``run_exchange`` (materialized, identity expert,
fp32 payloads from ``make_token_payloads(payload_seed)``, its f64 k-ascending
reduction) runs on routing from its own ``gen_realworld``; the script stores
sha256 digests of every rank's activation and output bytes and of
``row_of`` (int64, ``_activation_layouts``), plus the dedup ``loads``.  The
GPU test (tests/test_gpu_fullsize.py) regenerates the same routing and
payloads, runs the CUDA path and compares digests — parity pinned to the
reference itself at the contract sizes.
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

import shuffleforge as ref
from shuffleforge.planner import _activation_layouts

OUT = Path(__file__).resolve().parent / "digests.json"

# name: (P, experts, topk, tokens/rank, token_bytes, zipf_s, seed, payload_seed)
# BASELINE.json configs[0] is the oracle case; the others are the bf16
# configs' shapes with the reference's own fp32 payload rows of the same
# byte width (the descriptor path is byte-level).
CASES = {
    "oracle_2x4096_h1024_f32": (2, 8, 2, 4096, 4096, 0.0, 0, 0),
    "dsv3_decode_ep8": (8, 256, 8, 128, 14336, 0.0, 0, 0),
    "qwen3_ep8": (8, 128, 8, 4096, 4096, 0.0, 0, 0),
    "mixtral_ep2": (2, 8, 2, 8192, 8192, 0.0, 0, 0),
    "dsv3_zipf_ep4": (4, 256, 8, 4096, 14336, 1.2, 0, 0),
    "dsv3_ep8": (8, 256, 8, 4096, 14336, 0.0, 0, 0),
    "mixtral_ep8": (8, 8, 2, 8192, 8192, 0.0, 0, 0),
}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8).reshape(-1).data).hexdigest()


def make(name: str) -> dict:
    P, E, K, T_l, tb, zipf, seed, pseed = CASES[name]
    topo = ref.ClusterTopology(P, 1)
    pl = ref.round_robin_placement(E, topo)
    a = ref.gen_realworld(P * T_l, K, topo, pl, seed=seed, zipf_s=zipf)
    t0 = time.perf_counter()
    r = ref.run_exchange(a, topo, pl, tb, payload_seed=pseed)
    dt = time.perf_counter() - t0
    _, row_of = _activation_layouts(a, pl, topo)
    return {
        "P": P, "experts": E, "topk": K, "tokens_per_rank": T_l, "token_bytes": tb, "zipf_s": zipf,
        "seed": seed, "payload_seed": pseed,
        "row_of": sha(row_of.astype(np.int64)),
        "activation": [sha(r.activation(g)) for g in range(P)],
        "act_rows": [int(r.activation(g).size // tb) for g in range(P)],
        "output": [sha(r.output(s)) for s in range(P)],
        "loads": [int(x) for x in ref.dispatch_loads(a, pl, topo, tb)],
        "reference_s": round(dt, 2),
    }


if __name__ == "__main__":
    doc = json.loads(OUT.read_text()) if OUT.exists() else {}
    for name in sys.argv[1:] or CASES:
        doc[name] = make(name)
        print(name, doc[name]["reference_s"], "s", flush=True)
        OUT.write_text(json.dumps(doc, indent=1, sort_keys=True) + "\n")
