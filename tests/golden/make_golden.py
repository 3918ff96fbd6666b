"""Generate golden fixtures from the reference implementation itself.

Run in the build container (the reference is importable there, not on the
GPU box):

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Each case runs the reference ``run_exchange`` (materialized) plus its
planner helpers and stores routing inputs and every artefact the GPU path
must reproduce: activation bytes per rank, outputs per rank, row_of
(``_activation_layouts``), first_mask (``derive_token_node``) and
``dispatch_loads``.  Payloads are regenerated from ``payload_seed``.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

import shuffleforge as ref
from shuffleforge.engine import identity_expert, scaled_expert
from shuffleforge.planner import _activation_layouts
from shuffleforge.routing import derive_token_node

OUT = Path(__file__).resolve().parent

# name: (num_nodes, gpus_per_node, experts, topk, tokens, token_bytes, generator, kwargs, seed, expert)
CASES = {
    "box2_e8k2_uniform": (2, 1, 8, 2, 512, 64, "realworld", {"zipf_s": 0.0}, 0, "identity"),
    "box8_e256k8_zipf": (8, 1, 256, 8, 512, 128, "realworld", {"zipf_s": 1.2}, 0, "identity"),
    "box8_e64k8_scaled": (8, 1, 64, 8, 256, 96, "realworld", {"zipf_s": 1.1}, 2, "scaled"),
    "box4_single_node": (4, 1, 16, 4, 200, 32, "single_node", {"remote_only": True}, 4, "identity"),
    "grid4x4_e32k4": (4, 4, 32, 4, 96, 64, "realworld", {}, 3, "identity"),
    "grid2x2_imbalanced": (2, 2, 16, 2, 300, 48, "imbalanced", {}, 5, "scaled"),
    "box1_degenerate": (1, 1, 1, 1, 16, 16, "realworld", {}, 6, "identity"),
    "box3_ragged_tb12": (3, 1, 9, 3, 100, 12, "realworld", {"zipf_s": 0.5}, 7, "identity"),
}


def make(name: str) -> None:
    n, m, E, K, T, tb, gen, kw, seed, expert = CASES[name]
    topo = ref.ClusterTopology(n, m)
    pl = ref.round_robin_placement(E, topo)
    gfn = {"realworld": ref.gen_realworld, "single_node": ref.gen_single_node,
           "imbalanced": ref.gen_imbalanced}[gen]
    a = gfn(T, K, topo, pl, seed=seed, **kw)
    fn = scaled_expert(E) if expert == "scaled" else identity_expert
    payload_seed = seed + 100
    r = ref.run_exchange(a, topo, pl, tb, payload_seed=payload_seed, expert_fn=fn)
    P = topo.num_gpus
    _, row_of = _activation_layouts(a, pl, topo)
    acts = [r.activation(g) for g in range(P)]
    outs = [r.output(s) for s in range(P)]
    lay = r.dispatch_plan.layouts
    np.savez_compressed(
        OUT / f"{name}.npz",
        num_nodes=n, gpus_per_node=m, num_experts=E, topk=K, token_bytes=tb, payload_seed=payload_seed,
        expert=np.array(expert), experts=a.experts, weights=a.weights, source=a.source, owner=pl.owner,
        row_of=row_of, first_mask=derive_token_node(a, pl, topo).first_mask,
        loads=ref.dispatch_loads(a, pl, topo, tb),
        act_rows=np.array([x.size // tb for x in acts]), activations=np.concatenate(acts),
        out_rows=np.array([x.size // tb for x in outs]), outputs=np.concatenate(outs),
        lay_expert_ids=np.concatenate([lay[g].expert_ids for g in range(P)]),
        lay_token_ids=np.concatenate([lay[g].token_ids for g in range(P)]),
        lay_k_col=np.concatenate([lay[g].k_col for g in range(P)]),
    )


if __name__ == "__main__":
    for name in sys.argv[1:] or CASES:
        make(name)
        print("wrote", OUT / f"{name}.npz")
