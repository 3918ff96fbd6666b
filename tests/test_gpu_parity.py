"""Parity of the sm_100a path with the reference (golden vectors) and the
oracle, on one B200 with P ranks emulated (every kernel addresses its
"peers" through the same pointer table it uses over NVLink).

Bars: layout metadata and dispatched activations bit-exact; combine
bit-exact in f64-accumulate mode, and within the stated tolerance in the
production fp32-accumulate mode (fp32 payloads rtol 1e-5 / atol 1e-6, the
reference's own criterion-1 bound, test_acceptance.py:91; bf16 payloads
rtol 2^-8 / atol 1e-3)."""

import numpy as np
import pytest

from conftest import golden_names, load_golden, split_rows
from oracle import shuffle_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

F32_TOL = dict(rtol=1e-5, atol=1e-6)
BF16_TOL = dict(rtol=2.0**-8, atol=1e-3)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2512_22036_b200 import _lib

    _lib.load()  # loud failure if the extension is missing
    torch.cuda.set_device(0)


def _pkg():
    import paper_2512_22036_b200 as pkg

    return pkg


# ---------------------------------------------------------------------------
# golden vectors written by the reference


@pytest.mark.parametrize("name", golden_names())
def test_run_exchange_matches_reference_golden(name):
    pkg = _pkg()
    g = load_golden(name)
    topo = pkg.ClusterTopology(g["num_nodes"], g["gpus_per_node"])
    pl = pkg.ExpertPlacement(g["num_experts"], g["owner"])
    a = pkg.RoutingAssignment(g["experts"].shape[0], g["topk"], g["experts"], g["weights"], g["source"])
    fn = pkg.scaled_expert(g["num_experts"]) if g["expert"] == "scaled" else pkg.identity_expert
    r = pkg.run_exchange(a, topo, pl, g["token_bytes"], payload_seed=g["payload_seed"], expert_fn=fn)
    P = topo.num_gpus
    tb = g["token_bytes"]
    acts = split_rows(g["activations"], g["act_rows"], tb)
    outs = split_rows(g["outputs"], g["out_rows"], tb)
    for rank in range(P):
        assert np.array_equal(r.activation(rank).reshape(-1, tb), acts[rank]), f"activation/{rank}"
        assert np.array_equal(r.output(rank).reshape(-1, tb), outs[rank]), f"output/{rank}"
    assert np.array_equal(r.dispatch_plan.row_of, g["row_of"])
    assert np.array_equal(r.dispatch_plan.first_mask, g["first_mask"])
    assert np.array_equal(r.dispatch_plan.loads, g["loads"])
    lay_t = np.concatenate([r.dispatch_plan.layouts[q].token_ids for q in range(P)])
    lay_k = np.concatenate([r.dispatch_plan.layouts[q].k_col for q in range(P)])
    assert np.array_equal(lay_t, g["lay_token_ids"]) and np.array_equal(lay_k, g["lay_k_col"])
    assert r.dispatch_report.rearrange_bytes == 0 and r.combine_report.rearrange_bytes == 0


def test_run_exchange_fp32_accumulate_within_reference_tolerance():
    pkg = _pkg()
    g = load_golden("box8_e256k8_zipf")
    topo = pkg.ClusterTopology(g["num_nodes"], g["gpus_per_node"])
    pl = pkg.ExpertPlacement(g["num_experts"], g["owner"])
    a = pkg.RoutingAssignment(g["experts"].shape[0], g["topk"], g["experts"], g["weights"], g["source"])
    r = pkg.run_exchange(a, topo, pl, g["token_bytes"], payload_seed=g["payload_seed"], acc="f32")
    tb = g["token_bytes"]
    outs = split_rows(g["outputs"], g["out_rows"], tb)
    for s in range(topo.num_gpus):
        got = r.output(s).view(np.float32)
        want = outs[s].reshape(-1).view(np.float32)
        np.testing.assert_allclose(got, want, **F32_TOL)
    # identity experts: the round trip reproduces the tokens (criterion 1)
    src = r.payloads.view(np.float32).reshape(a.num_tokens, -1)
    for s in range(topo.num_gpus):
        ids = r.combine_plan.local_tokens[s]
        np.testing.assert_allclose(r.output_f32(s), src[ids], **F32_TOL)


# ---------------------------------------------------------------------------
# oracle parity at DSV3 / Qwen3 / Mixtral shapes (bf16 payloads)


def _cluster_case(P, E, K, T_l, hidden, dtype, zipf, seed, max_tokens=None):
    pkg = _pkg()
    topo = pkg.box(P)
    pl = pkg.round_robin_placement(E, topo)
    a = pkg.gen_realworld(P * T_l, K, topo, pl, seed=seed, zipf_s=zipf)
    elem = 2 if dtype == "bf16" else 4
    tb = hidden * elem
    rng = np.random.default_rng(seed + 1)
    vals = rng.standard_normal((a.num_tokens, hidden)).astype(np.float32)
    payload = O.encode(vals, dtype)  # [T, tb] bytes
    return pkg, topo, pl, a, tb, payload


def _run_cluster(pkg, topo, pl, a, tb, payload, dtype, acc, cl=None, w_at_dispatch=None):
    """One emulated shuffle.  The router weights go to the dispatch too
    (fs_dispatch_w) for fp32 accumulation by default, so the f32 results
    cover the owner-side pre-reduction path wherever a token has >= 3 rows
    (>= 2 for fp32 rows) on one remote owner."""
    from paper_2512_22036_b200.engine import EmulatedCluster, dtype_code

    P = topo.num_gpus
    tdt, code = dtype_code(dtype)
    ids = [np.flatnonzero(a.source == s) for s in range(P)]
    own = cl is None
    if own:
        cl = EmulatedCluster(P, pl.num_experts, a.topk, tb, max(i.size for i in ids), owner=pl.owner)
    dev = cl.device
    idx = [torch.as_tensor(a.experts[i], device=dev) for i in ids]
    w = [torch.as_tensor(a.weights[i], dtype=torch.float64 if acc == "f64" else torch.float32, device=dev)
         for i in ids]
    xs = [torch.as_tensor(payload[i], device=dev).contiguous() for i in ids]
    plans = cl.layout(idx)
    if w_at_dispatch is None:
        w_at_dispatch = acc == "f32"
    cl.dispatch(xs, plans, ws=w if w_at_dispatch else None)
    outs = [torch.empty((i.size, tb), dtype=torch.uint8, device=dev) for i in ids]
    cl.combine(plans, w, [o.view(tdt) for o in outs], dtype_code=code, acc=1 if acc == "f64" else 0)
    cl.check()
    acts = [cl.ranks[s].act(plans[s].num_rows).cpu().numpy() for s in range(P)]
    res = dict(
        row_of=[p.row_of.cpu().numpy() for p in plans],
        counts=[p.expert_counts.cpu().numpy() for p in plans],
        offsets=[p.expert_offsets.cpu().numpy() for p in plans],
        stats=[p.stats.cpu().numpy() for p in plans],
        first=[p.first_mask.cpu().numpy() for p in plans],
        rank_mask=[p.rank_mask.cpu().numpy() for p in plans],
        acts=acts,
        outs=[o.cpu().numpy() for o in outs],
        ids=ids,
    )
    if own:
        cl.close()
    return res


def _check_layout(res, a, pl, P):
    layouts, row_of = O.activation_layouts(a.experts, a.source, pl.owner, P)
    fm = O.first_mask(a.experts, pl.owner, 1)
    dedup = O.dispatch_loads(a.experts, a.source, pl.owner, P, 1, 1)
    for s in range(P):
        ids = res["ids"][s]
        assert np.array_equal(res["row_of"][s], row_of[ids]), f"row_of rank {s}"
        assert np.array_equal(res["first"][s].astype(bool), fm[ids])
        loc = np.flatnonzero(pl.owner == s)
        cnt = np.array([(a.experts == e).sum() for e in loc])
        assert np.array_equal(res["counts"][s], cnt)
        assert np.array_equal(res["offsets"][s], np.concatenate(([0], np.cumsum(cnt))))
        st = res["stats"][s]
        assert st[0] == layouts[s].num_rows
        assert st[1] == dedup[s] and st[4] == dedup[s]
        own = pl.owner[a.experts[ids]]
        assert st[2] == int((own != s).sum()) and st[3] == int((own == s).sum())
        rm = np.zeros(ids.size, dtype=np.int64)
        for k in range(a.topk):
            rm |= 1 << own[:, k]
        assert np.array_equal(res["rank_mask"][s].astype(np.int64) & 0xFFFFFFFF, rm)
    return layouts, row_of


@pytest.mark.parametrize(
    "P,E,K,T_l,hidden,zipf",
    [
        (8, 256, 8, 256, 7168, 0.0),   # DeepSeek-V3 shape, uniform
        (8, 256, 8, 128, 7168, 1.2),   # DeepSeek-V3 decode batch, Zipf-skewed
        (8, 128, 8, 512, 2048, 0.0),   # Qwen3-30B-A3B shape
        (4, 8, 2, 1024, 4096, 0.0),    # Mixtral shape, EP=4
        (2, 8, 2, 1024, 4096, 1.2),    # Mixtral shape, EP=2, skewed
        (1, 8, 2, 2048, 4096, 0.0),    # single GPU: local permutation
    ],
)
def test_bf16_parity_with_oracle(P, E, K, T_l, hidden, zipf):
    pkg, topo, pl, a, tb, payload = _cluster_case(P, E, K, T_l, hidden, "bf16", zipf, seed=P * 7 + K)
    res64 = _run_cluster(pkg, topo, pl, a, tb, payload, "bf16", "f64")
    layouts, row_of = _check_layout(res64, a, pl, P)
    acts = O.dispatch(payload, layouts)
    for g in range(P):
        assert np.array_equal(res64["acts"][g], acts[g]), f"activation/{g}"
    for s in range(P):
        want = O.combine(acts, row_of, a.experts, a.weights, pl.owner, res64["ids"][s], "bf16")
        assert np.array_equal(res64["outs"][s], want), f"f64-accumulate output/{s} not bit-exact"
    res32 = _run_cluster(pkg, topo, pl, a, tb, payload, "bf16", "f32")
    for s in range(P):
        want = O.decode(O.combine(acts, row_of, a.experts, a.weights, pl.owner, res64["ids"][s], "bf16"), "bf16")
        got = O.decode(res32["outs"][s], "bf16")
        np.testing.assert_allclose(got, want, **BF16_TOL)


ENGINES = [("warp", "warp"), ("tma", "tma"), ("tma", "warp"), ("warp", "tma")]


@pytest.fixture(params=ENGINES, ids=lambda e: f"dispatch-{e[0]}_combine-{e[1]}")
def engines(request, monkeypatch):
    """Select the dispatch / combine data movers for handles created in the test."""
    monkeypatch.setenv("FUSCO_DISPATCH", request.param[0])
    monkeypatch.setenv("FUSCO_COMBINE", request.param[1])
    yield request.param


@pytest.mark.parametrize(
    "P,E,K,T_l,hidden,zipf",
    [
        (8, 256, 8, 128, 7168, 1.2),
        (4, 8, 2, 1024, 4096, 0.0),
        (1, 8, 2, 2048, 4096, 0.0),
        (2, 16, 4, 333, 1024, 0.3),
        (8, 64, 8, 64, 512, 0.0),
    ],
)
def test_engine_parity_with_oracle(engines, P, E, K, T_l, hidden, zipf):
    pkg, topo, pl, a, tb, payload = _cluster_case(P, E, K, T_l, hidden, "bf16", zipf, seed=P * 5 + K)
    res = _run_cluster(pkg, topo, pl, a, tb, payload, "bf16", "f64")
    layouts, row_of = _check_layout(res, a, pl, P)
    acts = O.dispatch(payload, layouts)
    for g in range(P):
        assert np.array_equal(res["acts"][g], acts[g]), f"activation/{g}"
    for s in range(P):
        want = O.combine(acts, row_of, a.experts, a.weights, pl.owner, res["ids"][s], "bf16")
        assert np.array_equal(res["outs"][s], want), f"output/{s}"
    res32 = _run_cluster(pkg, topo, pl, a, tb, payload, "bf16", "f32")
    for s in range(P):
        want = O.decode(O.combine(acts, row_of, a.experts, a.weights, pl.owner, res["ids"][s], "bf16"), "bf16")
        np.testing.assert_allclose(O.decode(res32["outs"][s], "bf16"), want, **BF16_TOL)


@pytest.mark.parametrize("slices", [0, 1, 3, 7])
@pytest.mark.parametrize("P,E,K,T_l,hidden", [(1, 256, 8, 700, 7168), (1, 8, 2, 1500, 4096),
                                             (4, 32, 4, 300, 1032)])
def test_tma_dispatch_column_slices(monkeypatch, slices, P, E, K, T_l, hidden):
    """The TMA dispatch's work unit is a whole row or a (token, column slice):
    slices=0 slices only the last partial round of the grid (FUSCO_TMA_TAIL=1),
    n > 0 slices every row (odd n leaves a shorter last slice).  At P > 1
    block completion counts units, not tokens.  Activations and the combine
    stay bit-exact."""
    monkeypatch.setenv("FUSCO_DISPATCH", "tma")
    if slices:
        monkeypatch.setenv("FUSCO_TMA_SLICES", str(slices))
    else:
        monkeypatch.setenv("FUSCO_TMA_TAIL", "1")
    pkg, topo, pl, a, tb, payload = _cluster_case(P, E, K, T_l, hidden, "bf16", 0.9, seed=31 + slices)
    res = _run_cluster(pkg, topo, pl, a, tb, payload, "bf16", "f64")
    layouts, row_of = _check_layout(res, a, pl, P)
    acts = O.dispatch(payload, layouts)
    for g in range(P):
        assert np.array_equal(res["acts"][g], acts[g]), f"activation/{g}"
    for s in range(P):
        want = O.combine(acts, row_of, a.experts, a.weights, pl.owner, res["ids"][s], "bf16")
        assert np.array_equal(res["outs"][s], want), f"output/{s}"


@pytest.mark.parametrize("P,E,K,T_l,hidden", [(4, 8, 2, 1024, 4096), (8, 256, 8, 128, 7168), (2, 16, 4, 333, 1024)])
def test_push_rounds_parity(monkeypatch, P, E, K, T_l, hidden):
    """Per-CTA-round completion counting (FUSCO_PUSH_ROUNDS=1, the A/B variant
    of the per-unit count): same layout, activations and combine, bit-exact."""
    monkeypatch.setenv("FUSCO_DISPATCH", "warp")
    monkeypatch.setenv("FUSCO_PUSH_ROUNDS", "1")
    pkg, topo, pl, a, tb, payload = _cluster_case(P, E, K, T_l, hidden, "bf16", 0.5, seed=77 + P)
    res = _run_cluster(pkg, topo, pl, a, tb, payload, "bf16", "f64")
    layouts, row_of = _check_layout(res, a, pl, P)
    acts = O.dispatch(payload, layouts)
    for g in range(P):
        assert np.array_equal(res["acts"][g], acts[g]), f"activation/{g}"
    for s in range(P):
        want = O.combine(acts, row_of, a.experts, a.weights, pl.owner, res["ids"][s], "bf16")
        assert np.array_equal(res["outs"][s], want), f"output/{s}"


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("P,E,K,T_l,hidden,zipf", [(2, 16, 8, 700, 1024, 0.0), (4, 64, 8, 300, 2048, 1.2),
                                                    (8, 256, 8, 128, 7168, 1.2), (3, 12, 4, 257, 520, 0.5)])
def test_owner_reduce_parity(monkeypatch, dtype, P, E, K, T_l, hidden, zipf):
    """Owner-side pre-reduction (weights at dispatch, fp32 accumulate): within
    the stated tolerance of the oracle and of the plain pull combine; the
    activations stay bit-exact; weights at dispatch with f64 accumulation stay
    bit-exact (no pre-reduction on that path)."""
    monkeypatch.setenv("FUSCO_DISPATCH", "warp")
    monkeypatch.setenv("FUSCO_COMBINE", "tma")
    monkeypatch.setenv("FUSCO_OWNER_REDUCE", "1")  # at every world size and batch (default: P = 2, > 512 tokens)
    pkg, topo, pl, a, tb, payload = _cluster_case(P, E, K, T_l, hidden, dtype, zipf, seed=500 + P)
    red = _run_cluster(pkg, topo, pl, a, tb, payload, dtype, "f32", w_at_dispatch=True)
    plain = _run_cluster(pkg, topo, pl, a, tb, payload, dtype, "f32", w_at_dispatch=False)
    exact = _run_cluster(pkg, topo, pl, a, tb, payload, dtype, "f64", w_at_dispatch=True)
    layouts, row_of = _check_layout(red, a, pl, P)
    acts = O.dispatch(payload, layouts)
    tol = BF16_TOL if dtype == "bf16" else dict(rtol=1e-5, atol=1e-6)
    mmin = 3 if dtype == "bf16" else 2
    grouped = 0
    for s in range(P):
        ids = red["ids"][s]
        owners = pl.owner[a.experts[ids]]
        for g in range(P):
            if g != s:
                grouped += int(((owners == g).sum(axis=1) >= mmin).sum())
        want_b = O.combine(acts, row_of, a.experts, a.weights, pl.owner, ids, dtype)
        assert np.array_equal(exact["outs"][s], want_b), f"f64 output/{s} with weights at dispatch"
        want = O.decode(want_b, dtype)
        np.testing.assert_allclose(O.decode(red["outs"][s], dtype), want, **tol)
        np.testing.assert_allclose(O.decode(red["outs"][s], dtype), O.decode(plain["outs"][s], dtype), **tol)
    for g in range(P):
        assert np.array_equal(red["acts"][g], acts[g]), f"activation/{g}"
    assert grouped > 0, "the case must exercise pre-reduced groups"


def test_owner_reduce_ragged_mixed_decisions(monkeypatch):
    """P = 2 with 700 tokens on rank 0 and 300 on rank 1: by default only
    rank 0 pre-reduces as an owner (> 512 tokens), rank 1 does not; each
    source pulls partials only from owners whose mode word says so.  Both
    outputs within tolerance, activations bit-exact, over two epochs."""
    from paper_2512_22036_b200.engine import EmulatedCluster

    monkeypatch.setenv("FUSCO_DISPATCH", "warp")
    monkeypatch.setenv("FUSCO_COMBINE", "tma")
    monkeypatch.delenv("FUSCO_OWNER_REDUCE", raising=False)
    P, E, K, hidden = 2, 16, 8, 1024
    pkg = _pkg()
    topo = pkg.box(P)
    pl = pkg.round_robin_placement(E, topo)
    a = pkg.gen_realworld(P * 700, K, topo, pl, seed=91, zipf_s=0.3)
    ids = [np.flatnonzero(a.source == 0)[:700], np.flatnonzero(a.source == 1)[:300]]
    sel = np.sort(np.concatenate(ids))
    experts, weights, source = a.experts[sel], a.weights[sel], a.source[sel]
    loc = [np.flatnonzero(source == s) for s in range(P)]
    tb = hidden * 2
    vals = np.random.default_rng(5).standard_normal((sel.size, hidden)).astype(np.float32)
    payload = O.encode(vals, "bf16")
    layouts, row_of = O.activation_layouts(experts, source, pl.owner, P)
    acts = O.dispatch(payload, layouts)
    with EmulatedCluster(P, E, K, tb, 700, owner=pl.owner) as cl:
        dev = cl.device
        idx = [torch.as_tensor(experts[i], device=dev) for i in loc]
        xs = [torch.as_tensor(payload[i], device=dev).contiguous() for i in loc]
        ws = [torch.as_tensor(weights[i], dtype=torch.float32, device=dev) for i in loc]
        for _ in range(2):
            plans = cl.layout(idx)
            cl.dispatch(xs, plans, ws=ws)
            outs = [torch.empty((i.size, tb), dtype=torch.uint8, device=dev) for i in loc]
            cl.combine(plans, ws, [o.view(torch.bfloat16) for o in outs], dtype_code=1, acc=0)
            cl.check()
            for g in range(P):
                assert np.array_equal(cl.ranks[g].act(plans[g].num_rows).cpu().numpy(), acts[g])
            for s_ in range(P):
                want = O.decode(O.combine(acts, row_of, experts, weights, pl.owner, loc[s_], "bf16"), "bf16")
                np.testing.assert_allclose(O.decode(outs[s_].cpu().numpy(), "bf16"), want, **BF16_TOL)


def test_engine_parity_fp32_payload(engines):
    """fp32 rows (the reference's own payload dtype) through both engines."""
    pkg, topo, pl, a, tb, payload = _cluster_case(4, 32, 4, 300, 1024, "f32", 0.7, seed=9)
    res = _run_cluster(pkg, topo, pl, a, tb, payload, "f32", "f64")
    layouts, row_of = _check_layout(res, a, pl, 4)
    acts = O.dispatch(payload, layouts)
    for s in range(4):
        assert np.array_equal(res["acts"][s], acts[s])
        want = O.combine(acts, row_of, a.experts, a.weights, pl.owner, res["ids"][s], "f32")
        assert np.array_equal(res["outs"][s], want)


def test_repeated_epochs_reuse_buffers():
    """Four consecutive shuffles on one cluster (epoch parity flips the
    double-buffered activation/count/fan-out regions)."""
    from paper_2512_22036_b200.engine import EmulatedCluster

    P, E, K, T_l, hidden = 4, 32, 4, 200, 512
    pkg = _pkg()
    cl = EmulatedCluster(P, E, K, hidden * 2, T_l, owner=np.arange(E) % P)
    try:
        for it in range(4):
            _, topo, pl, a, tb, payload = _cluster_case(P, E, K, T_l, hidden, "bf16", 0.6 * it, seed=100 + it)
            res = _run_cluster(pkg, topo, pl, a, tb, payload, "bf16", "f64", cl=cl)
            layouts, row_of = _check_layout(res, a, pl, P)
            acts = O.dispatch(payload, layouts)
            for g in range(P):
                assert np.array_equal(res["acts"][g], acts[g])
            for s in range(P):
                want = O.combine(acts, row_of, a.experts, a.weights, pl.owner, res["ids"][s], "bf16")
                assert np.array_equal(res["outs"][s], want)
    finally:
        cl.close()


def test_mixtral_full_size_single_gpu_properties():
    """BASELINE configs[1] at full size on one GPU (8192 tokens, hidden 4096
    bf16, 8 experts top-2): size-independent properties instead of the
    oracle — every activation row is its token's row (a permutation with
    K-fold fan-out), counts sum to T*K, and the identity round trip returns
    Σ_k w_k·x = x (weights sum to 1) within bf16 tolerance."""
    from paper_2512_22036_b200.engine import EmulatedCluster

    pkg = _pkg()
    T, E, K, H = 8192, 8, 2, 4096
    topo = pkg.box(1)
    pl = pkg.round_robin_placement(E, topo)
    a = pkg.gen_realworld(T, K, topo, pl, seed=0, zipf_s=0.0)
    dev = torch.device("cuda", 0)
    x = torch.randn(T, H, device=dev).to(torch.bfloat16)
    idx = torch.as_tensor(a.experts, device=dev)
    w = torch.as_tensor(a.weights, dtype=torch.float32, device=dev)
    with EmulatedCluster(1, E, K, H * 2, T) as cl:
        plans = cl.layout([idx])
        cl.dispatch([x], plans)
        out = torch.empty_like(x)
        cl.combine(plans, [w], [out], dtype_code=1)
        cl.check()
        p = plans[0]
        rows = p.num_rows
        assert rows == T * K and int(p.expert_counts.sum()) == T * K
        act = cl.ranks[0].act(rows, torch.bfloat16)
        tok = torch.empty(rows, dtype=torch.int64, device=dev)
        tok[p.row_of.reshape(-1).long()] = torch.arange(T, device=dev).repeat_interleave(K)
        assert torch.equal(act, x[tok])
        # expert-major: rows of expert e are contiguous and sorted by token
        eid = torch.empty(rows, dtype=torch.int64, device=dev)
        eid[p.row_of.reshape(-1).long()] = idx.reshape(-1)
        assert bool((eid[1:] >= eid[:-1]).all())
        same = eid[1:] == eid[:-1]
        assert bool((tok[1:][same] > tok[:-1][same]).all())
        ref = (x.float() * w.sum(1, keepdim=True)).to(torch.bfloat16).float()
        torch.testing.assert_close(out.float(), ref, rtol=2.0**-7, atol=2e-2)


def test_empty_rank_and_zero_tokens():
    pkg = _pkg()
    topo = pkg.box(3)
    pl = pkg.round_robin_placement(6, topo)
    experts = np.array([[0, 1], [2, 4], [5, 3], [1, 2]])
    weights = np.full((4, 2), 0.5)
    source = np.array([0, 0, 2, 2])  # rank 1 has no tokens
    a = pkg.RoutingAssignment(4, 2, experts, weights, source)
    r = pkg.run_exchange(a, topo, pl, 64, payload_seed=1)
    res = O.exchange(experts, weights, source, pl.owner, 3, r.payloads)
    for g in range(3):
        assert np.array_equal(r.activation(g), res["activations"][g].reshape(-1))
        assert np.array_equal(r.output(g), res["outputs"][g].reshape(-1))


def test_device_errors_raise_value_error():
    from paper_2512_22036_b200.engine import EmulatedCluster

    with EmulatedCluster(2, 8, 2, 64, 16) as cl:
        dev = cl.device
        bad = [torch.tensor([[0, 9]], device=dev), torch.tensor([[1, 2]], device=dev)]  # expert 9 >= E
        cl.layout(bad)
        with pytest.raises(ValueError):
            cl.check()
        dup = [torch.tensor([[3, 3]], device=dev), torch.tensor([[1, 2]], device=dev)]
        cl.layout(dup)
        with pytest.raises(ValueError):
            cl.check()
        ok = [torch.tensor([[0, 1]], device=dev), torch.tensor([[1, 2]], device=dev)]
        cl.layout(ok)
        cl.check()


def test_disaggregated_baseline_single_gpu_matches_fused():
    """§8f next row: the pack/all-to-all/unpack baseline lands the same bytes."""
    from paper_2512_22036_b200.baseline import DisaggregatedShuffle

    pkg, topo, pl, a, tb, payload = _cluster_case(1, 32, 4, 700, 1024, "bf16", 0.8, seed=21)
    res = _run_cluster(pkg, topo, pl, a, tb, payload, "bf16", "f64")
    dev = torch.device("cuda", 0)
    base = DisaggregatedShuffle(num_experts=32, topk=4, device=dev)
    x = torch.as_tensor(payload, device=dev).view(torch.bfloat16)
    act, st = base.dispatch(x, torch.as_tensor(a.experts, device=dev))
    assert np.array_equal(act.view(torch.uint8).cpu().numpy(), res["acts"][0])
    out = base.combine(act, st, torch.as_tensor(a.weights, dtype=torch.float32, device=dev))
    np.testing.assert_allclose(out.float().cpu().numpy(), O.decode(res["outs"][0], "bf16"), **BF16_TOL)
    assert base.rearrange_bytes(700, 4, tb) == 4 * 700 * 4 * tb


@pytest.mark.parametrize("planner", ["cluster", "grid"])
@pytest.mark.parametrize("E,K,T,zipf", [(8, 2, 8192, 0.0), (256, 8, 4096, 1.2), (64, 4, 1000, 0.5), (16, 3, 1, 0.0),
                                        (256, 8, 7777, 0.0), (512, 8, 600, 0.0), (32, 12, 300, 0.0)])
def test_planner_engines_single_rank(monkeypatch, planner, E, K, T, zipf):
    """One-cluster DSMEM planner (E <= 256, K <= 8, T <= 8192) and the grid
    planner give the reference layout (larger E/K fall back to the grid one)."""
    monkeypatch.setenv("FUSCO_LAYOUT", planner)
    from paper_2512_22036_b200.engine import EmulatedCluster

    pkg = _pkg()
    topo = pkg.box(1)
    pl = pkg.round_robin_placement(E, topo)
    a = pkg.gen_realworld(T, K, topo, pl, seed=E + K, zipf_s=zipf)
    dev = torch.device("cuda", 0)
    with EmulatedCluster(1, E, K, 64, T) as cl:
        plans = cl.layout([torch.as_tensor(a.experts, device=dev)])
        cl.check()
        res = dict(row_of=[plans[0].row_of.cpu().numpy()], counts=[plans[0].expert_counts.cpu().numpy()],
                   offsets=[plans[0].expert_offsets.cpu().numpy()], stats=[plans[0].stats.cpu().numpy()],
                   first=[plans[0].first_mask.cpu().numpy()], rank_mask=[plans[0].rank_mask.cpu().numpy()],
                   ids=[np.arange(T)])
    _check_layout(res, a, pl, 1)


@pytest.mark.parametrize("ablate", [("planner",), ("balancer",), ("dcomm",), ("planner", "dcomm")])
@pytest.mark.parametrize("name", ["box8_e64k8_scaled", "grid2x2_imbalanced", "box2_e8k2_uniform"])
def test_run_exchange_ablations_match_reference_golden(name, ablate):
    """Reference ablations (engine.py:384-420): same bytes, different traffic
    (no dedup / disaggregated rearrangement passes / static groups)."""
    pkg = _pkg()
    g = load_golden(name)
    topo = pkg.ClusterTopology(g["num_nodes"], g["gpus_per_node"])
    pl = pkg.ExpertPlacement(g["num_experts"], g["owner"])
    a = pkg.RoutingAssignment(g["experts"].shape[0], g["topk"], g["experts"], g["weights"], g["source"])
    fn = pkg.scaled_expert(g["num_experts"]) if g["expert"] == "scaled" else pkg.identity_expert
    r = pkg.run_exchange(a, topo, pl, g["token_bytes"], payload_seed=g["payload_seed"], expert_fn=fn, ablate=ablate)
    tb = g["token_bytes"]
    acts = split_rows(g["activations"], g["act_rows"], tb)
    outs = split_rows(g["outputs"], g["out_rows"], tb)
    for rank in range(topo.num_gpus):
        assert np.array_equal(r.activation(rank).reshape(-1, tb), acts[rank])
        assert np.array_equal(r.output(rank).reshape(-1, tb), outs[rank])
    naive = pkg.naive_inter_node_bytes(a, pl, topo, tb)
    if "planner" in ablate or "dcomm" in ablate:
        assert r.dispatch_report.inter_node_bytes == naive
    if "dcomm" in ablate:
        assert r.dispatch_report.rearrange_bytes + r.combine_report.rearrange_bytes == 4 * a.num_tokens * a.topk * tb
    else:
        assert r.dispatch_report.rearrange_bytes == 0


@pytest.mark.gpu
def test_bench_matrix_rows_on_gpu():
    """§8f next row #2: every variant of a small matrix runs on the GPU and
    yields schema-valid rows; the planner-off and baseline variants move at
    least as many link bytes as the fused one (no dedup), the baseline
    reports its standalone rearrangement bytes (4·T·K·tb)."""
    from paper_2512_22036_b200 import matrix as M

    topo, pl = _pkg().preset("test")
    cfg = M.BenchConfig(topo, pl, ("realworld",), (512,), topk=4, token_bytes=256, repeats=1,
                        variants=tuple(M.VARIANT_ABLATE))
    doc = M.run_matrix(cfg)
    M.validate_result(doc)
    rows = {r["variant"]: r for r in doc["rows"]}
    assert set(rows) == set(M.VARIANT_ABLATE)
    for r in rows.values():
        assert r["total_s"] > 0 and r["latency_us"] > 0
        assert r["mode"] == ("gpu-eager" if r["variant"] in ("baseline", "dcomm_off") else "gpu-graph")
    assert rows["fused"]["rearrange_bytes"] == 0
    assert rows["baseline"]["rearrange_bytes"] == 4 * 512 * 4 * 256
    assert rows["planner_off"]["inter_node_bytes"] >= rows["fused"]["inter_node_bytes"]
    assert rows["fused"]["dedup_ratio"] >= 1.0


@pytest.mark.gpu
def test_bench_matrix_from_recorded_trace(tmp_path):
    """A captured routing drives the GPU matrix (--topology FILE --trace FILE)."""
    import json

    from paper_2512_22036_b200 import matrix as M

    pkg = _pkg()
    topo, pl = pkg.preset("test")
    a = pkg.gen_realworld(512, 4, topo, pl, seed=11, zipf_s=1.0)
    pkg.save_trace(tmp_path / "cap.json", a, 256)
    pkg.save_topology(tmp_path / "topo.json", topo, pl)
    out = tmp_path / "rows.json"
    assert M.main(["--topology", str(tmp_path / "topo.json"), "--trace", str(tmp_path / "cap.json"), "--variants",
                   "fused", "balancer_off", "--repeats", "1", "--format", "json", "--out", str(out)]) == 0
    doc = json.loads(out.read_text())
    M.validate_result(doc)
    assert [(r["pattern"], r["seq_len"], r["variant"]) for r in doc["rows"]] == [
        ("cap.json", 512, "fused"), ("cap.json", 512, "balancer_off")]
    assert doc["rows"][1]["balancer"] == "static"


@pytest.mark.gpu
@pytest.mark.parametrize("name", golden_names())
def test_device_plan_json_matches_oracle_plan(name):
    """§8f #4: the --dump-plan document of the device-built plans (layouts,
    per-(source, destination) transfers and local edges as descriptor wire
    blobs) is identical to the one derived from the reference layouts."""
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from test_host_api import _oracle_plans

    from paper_2512_22036_b200 import wire as W

    pkg = _pkg()
    g = load_golden(name)
    topo = pkg.ClusterTopology(g["num_nodes"], g["gpus_per_node"])
    pl = pkg.ExpertPlacement(int(g["num_experts"]), g["owner"])
    a = pkg.RoutingAssignment(g["experts"].shape[0], g["topk"], g["experts"], g["weights"], g["source"])
    d, c, _ = pkg.build_plan_pair(a, topo, pl, g["token_bytes"])
    od, oc, _, _ = _oracle_plans(g)
    m = g["gpus_per_node"]
    for got, want in ((W.plan_to_json(d, m), W.plan_to_json(od, m)), (W.plan_to_json(c, m), W.plan_to_json(oc, m))):
        for key in ("layouts", "node_transfers", "local_edges", "direction", "topk", "token_bytes"):
            assert got[key] == want[key], key


@pytest.mark.gpu
def test_ragged_epochs_stress(engines):
    """Twelve consecutive shuffles on one handle set with a different, ragged
    token count per rank every epoch (empty ranks, one-token ranks, full
    max_tokens batches, Zipf-skewed experts): every epoch bit-exact against
    the oracle — exercises the per-parity work counters, the done count with
    a work-sized grid, the fan-out list and the parity-buffered regions."""
    from paper_2512_22036_b200.engine import EmulatedCluster

    pkg = _pkg()
    P, E, K, hidden, T_max = 4, 32, 4, 256, 300
    topo = pkg.box(P)
    pl = pkg.round_robin_placement(E, topo)
    rng = np.random.default_rng(7)
    cl = EmulatedCluster(P, E, K, hidden * 2, T_max, owner=pl.owner)
    try:
        for it in range(12):
            counts = rng.integers(0, T_max + 1, size=P)
            counts[it % P] = (0, 1, T_max)[it % 3]
            T = int(counts.sum())
            if T == 0:
                counts[0], T = 1, 1
            base = pkg.gen_realworld(T, K, topo, pl, seed=200 + it, zipf_s=(0.0, 0.8, 1.4)[it % 3])
            source = np.repeat(np.arange(P), counts)
            a = pkg.RoutingAssignment(T, K, base.experts, base.weights, source)
            payload = O.encode(rng.standard_normal((T, hidden)).astype(np.float32), "bf16")
            res = _run_cluster(pkg, topo, pl, a, hidden * 2, payload, "bf16", "f64", cl=cl)
            layouts, row_of = _check_layout(res, a, pl, P)
            acts = O.dispatch(payload, layouts)
            for g in range(P):
                assert np.array_equal(res["acts"][g], acts[g]), f"epoch {it} activation/{g}"
            for s in range(P):
                want = O.combine(acts, row_of, a.experts, a.weights, pl.owner, res["ids"][s], "bf16")
                assert np.array_equal(res["outs"][s], want), f"epoch {it} output/{s}"
    finally:
        cl.close()


@pytest.mark.gpu
def test_missing_peer_times_out_loudly():
    """Failure detection: a rank whose peer never publishes its counts does not
    hang — the bounded flag wait records FS_ETIMEOUT and fs_check raises."""
    from paper_2512_22036_b200._lib import FS_ETIMEOUT, FS_PHASE_LOCAL, FS_PHASE_REMOTE, FuscoError
    from paper_2512_22036_b200.engine import EmulatedCluster

    P, E, K, T = 2, 8, 2, 64
    cl = EmulatedCluster(P, E, K, 256, T, owner=np.arange(E) % P, timeout_ms=200)
    try:
        r0 = cl.ranks[0]
        idx = torch.as_tensor(np.stack([np.arange(T) % E, (np.arange(T) + 1) % E], 1), device=cl.device)
        plan = r0.new_plan(idx)
        r0.layout(plan, FS_PHASE_LOCAL)
        r0.layout(plan, FS_PHASE_REMOTE)  # rank 1 never ran: its count words never arrive
        with pytest.raises(FuscoError) as ei:
            r0.check()
        assert ei.value.code == FS_ETIMEOUT
    finally:
        cl.close()


@pytest.mark.gpu
def test_cuda_graph_replay_with_captured_expert():
    """A CUDA graph that captures planner, dispatch, an expert reading the
    activation view, and combine replays correctly with fresh inputs every
    replay: the activation buffer lives at a fixed address (it is not
    double-buffered by epoch)."""
    pkg = _pkg()
    T, E, K, H = 256, 8, 2, 256
    buf = pkg.EPBuffer(num_experts=E, topk=K, hidden=H, dtype="f32", max_tokens=T, with_act_out=True)
    try:
        dev = buf.device
        topo = pkg.box(1)
        a = pkg.gen_realworld(T, K, topo, pkg.round_robin_placement(E, topo), seed=5)
        idx = torch.as_tensor(a.experts, device=dev)
        w = torch.as_tensor(a.weights, dtype=torch.float64, device=dev)
        x = torch.zeros((T, H), dtype=torch.float32, device=dev)
        out = torch.empty_like(x)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(side):
            with torch.cuda.graph(g, stream=side):
                plan = buf.build_plan(idx)
                act = buf.dispatch(x, plan)
                buf.expert_out().copy_(act * 2.0)  # the "expert": a captured torch kernel reading act
                buf.combine(plan, w, out, src="act_out", acc="f64")
        torch.cuda.current_stream().wait_stream(side)
        for it in range(4):
            x.copy_(torch.randn((T, H), generator=torch.Generator(device=dev).manual_seed(it), device=dev))
            g.replay()
            torch.cuda.synchronize()
            buf.check()
            torch.testing.assert_close(out, 2.0 * x, rtol=1e-6, atol=1e-6)
    finally:
        buf.close()
