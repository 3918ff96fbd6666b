"""The CPU oracle is pinned to the reference: golden vectors written by the
reference itself (tests/golden/make_golden.py), plus live cross-checks when
the reference is importable (this container only)."""

import numpy as np
import pytest

from conftest import golden_names, load_golden, split_rows
from oracle import shuffle_oracle as O


def _payloads(g):
    rng = np.random.default_rng(g["payload_seed"])
    tb = g["token_bytes"]
    vals = rng.standard_normal((g["experts"].shape[0], tb // 4)).astype(np.float32)
    return vals.view(np.uint8).reshape(-1, tb)


@pytest.mark.parametrize("name", golden_names())
def test_oracle_matches_golden(name):
    g = load_golden(name)
    P = g["num_nodes"] * g["gpus_per_node"]
    fn = O.scaled_expert if g["expert"] == "scaled" else O.identity_expert
    res = O.exchange(g["experts"], g["weights"], g["source"], g["owner"], P, _payloads(g), fn,
                     gpus_per_node=g["gpus_per_node"])
    tb = g["token_bytes"]
    acts = split_rows(g["activations"], g["act_rows"], tb)
    outs = split_rows(g["outputs"], g["out_rows"], tb)
    assert np.array_equal(res["row_of"], g["row_of"])
    assert np.array_equal(res["first_mask"], g["first_mask"])
    assert np.array_equal(res["loads"], g["loads"])
    for r in range(P):
        assert np.array_equal(res["activations"][r], acts[r])
        assert np.array_equal(res["outputs"][r], outs[r])
    lay_e = np.concatenate([res["layouts"][r].expert_ids for r in range(P)])
    lay_t = np.concatenate([res["layouts"][r].token_ids for r in range(P)])
    lay_k = np.concatenate([res["layouts"][r].k_col for r in range(P)])
    assert np.array_equal(lay_e, g["lay_expert_ids"])
    assert np.array_equal(lay_t, g["lay_token_ids"])
    assert np.array_equal(lay_k, g["lay_k_col"])


def test_descriptor_known_answers():
    """Descriptor semantics the GPU path implements with segment = one row
    (reference test_descriptor.py:31-65): gather [(8,4),(0,4)] of
    b'ABCDEFGHIJKL' -> b'IJKLABCD' is a row gather with 4-byte rows."""
    buf = np.frombuffer(b"ABCDEFGHIJKL", dtype=np.uint8).reshape(3, 4)
    lay = O.Layout(np.zeros(2, int), np.array([2, 0]), np.zeros(2, int), np.zeros(2, int))
    got = O.dispatch(buf, {0: lay})[0].tobytes()
    assert got == b"IJKLABCD"


def test_bf16_rounding_helpers():
    x = np.array([1.0, -2.5, 1 + 2**-8, 1 + 3 * 2**-9, 3.0e38, 1e-3], dtype=np.float64)
    # f64 -> bf16 must equal exact RNE: compare with a brute-force neighbour search
    b = O.f64_to_bf16(x)
    v = O.bf16_to_f32(b).astype(np.float64)
    for xi, vi, bi in zip(x, v, b):
        lo = O.bf16_to_f32(np.array([bi - 1], dtype=np.uint16))[0]
        hi = O.bf16_to_f32(np.array([bi + 1], dtype=np.uint16))[0]
        assert abs(vi - xi) <= abs(lo - xi) and abs(vi - xi) <= abs(hi - xi)
    # exact tie 1 + 2^-8 rounds to even (1.0)
    assert O.bf16_to_f32(O.f64_to_bf16(np.array([1 + 2**-8])))[0] == 1.0


def test_oracle_vs_live_reference_random(reference):
    ref = reference
    from shuffleforge.engine import scaled_expert

    rng = np.random.default_rng(77)
    for i in range(25):
        n, m = int(rng.choice([1, 2, 4])), int(rng.choice([1, 2, 4]))
        epg = int(rng.integers(1, 64 // (n * m) + 1))
        k = int(rng.integers(1, min(8, epg * m) + 1))
        T, tb = int(rng.integers(0, 400)), 4 * int(rng.integers(1, 17))
        topo = ref.ClusterTopology(n, m)
        pl = ref.round_robin_placement(n * m * epg, topo)
        a = ref.gen_realworld(T, k, topo, pl, seed=i, zipf_s=float(rng.choice([0.0, 1.2])))
        scaled = bool(i % 2)
        r = ref.run_exchange(a, topo, pl, tb, payload_seed=i,
                             expert_fn=scaled_expert(pl.num_experts) if scaled else ref.engine.identity_expert)
        res = O.exchange(a.experts, a.weights, a.source, pl.owner, topo.num_gpus, r.payloads,
                         O.scaled_expert if scaled else O.identity_expert, gpus_per_node=m)
        for g in range(topo.num_gpus):
            assert np.array_equal(res["activations"][g].reshape(-1), r.activation(g))
            assert np.array_equal(res["outputs"][g].reshape(-1), r.output(g))
        assert np.array_equal(res["loads"], ref.dispatch_loads(a, pl, topo, tb))
