"""Host-side logic (CPU only): the routing/topology/balancer mirrors agree
with the reference's golden inputs and known answers, and the C-ABI library
loads and exports every symbol include/fusco.h declares."""

import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, golden_names, load_golden
from paper_2512_22036_b200 import balancer as B
from paper_2512_22036_b200 import routing as R
from paper_2512_22036_b200 import topology as T

GEN_OF = {
    "box2_e8k2_uniform": ("realworld", {"zipf_s": 0.0}, 0),
    "box8_e256k8_zipf": ("realworld", {"zipf_s": 1.2}, 0),
    "box8_e64k8_scaled": ("realworld", {"zipf_s": 1.1}, 2),
    "box4_single_node": ("single_node", {"remote_only": True}, 4),
    "grid4x4_e32k4": ("realworld", {}, 3),
    "grid2x2_imbalanced": ("imbalanced", {}, 5),
    "box1_degenerate": ("realworld", {}, 6),
    "box3_ragged_tb12": ("realworld", {"zipf_s": 0.5}, 7),
}


@pytest.mark.parametrize("name", golden_names())
def test_generators_reproduce_reference_routing(name):
    g = load_golden(name)
    gen, kw, seed = GEN_OF[name]
    topo = T.ClusterTopology(g["num_nodes"], g["gpus_per_node"])
    pl = T.round_robin_placement(g["num_experts"], topo)
    a = R.GENERATORS[gen](g["experts"].shape[0], g["topk"], topo, pl, seed=seed, **kw)
    assert np.array_equal(a.experts, g["experts"])
    assert np.array_equal(a.weights, g["weights"])
    assert np.array_equal(a.source, g["source"])
    assert np.array_equal(pl.owner, g["owner"])
    assert np.array_equal(R.derive_token_node(a, pl, topo).first_mask, g["first_mask"])


def test_routing_validation_errors():
    with pytest.raises(ValueError):
        R.RoutingAssignment(1, 2, np.array([[3, 3]]), np.array([[0.5, 0.5]]), np.array([0]))
    with pytest.raises(ValueError):
        R.RoutingAssignment(1, 2, np.array([[1, 3]]), np.array([[0.7, 0.5]]), np.array([0]))
    with pytest.raises(ValueError):
        R.RoutingAssignment(1, 1, np.array([[-1]]), np.array([[1.0]]), np.array([0]))


def test_local_routing_and_sources():
    topo = T.box(4)
    pl = T.round_robin_placement(16, topo)
    a = R.gen_realworld(40, 2, topo, pl, seed=1)
    assert a.source.tolist() == [t % 4 for t in range(40)]
    ids, idx, w = R.local_routing(a, 2)
    assert ids.tolist() == list(range(2, 40, 4))
    assert np.array_equal(idx, a.experts[ids]) and np.array_equal(w, a.weights[ids])


def test_trace_round_trip(tmp_path):
    topo = T.box(2)
    pl = T.round_robin_placement(8, topo)
    a = R.gen_realworld(10, 2, topo, pl, seed=0)
    R.save_trace(tmp_path / "t.json", a, 64)
    b, tb = R.load_trace(tmp_path / "t.json")
    assert tb == 64 and np.array_equal(a.experts, b.experts) and np.array_equal(a.weights, b.weights)


def test_balancer_worked_example_and_rotation():
    """Reference test_balancer.py:49-57 (minimax 7) and heaviest GPU of node n in group n % M."""
    topo = T.ClusterTopology(2, 2)
    loads = np.array([[5, 3], [4, 1]])
    g = B.greedy_groups(loads, topo)
    assert B.group_load(loads, g, topo).max() == 7
    _, best = B.optimal_groups(loads, topo)
    assert best == 7
    rng = np.random.default_rng(0)
    for _ in range(50):
        topo = T.ClusterTopology(3, 4)
        L = rng.integers(0, 100, size=(3, 4))
        g = B.greedy_groups(L, topo)
        B.validate_groups(g, topo)
        for n in range(3):
            assert g[n, n % 4] == int(np.argsort(-L[n], kind="stable")[0])
    # inside one box (M = 1) the group table is trivial
    assert np.array_equal(B.greedy_groups(np.arange(8), T.box(8)), np.zeros((8, 1), dtype=np.int64))


def test_topology_json_and_presets(tmp_path):
    topo, pl = T.preset("large")
    assert topo.num_gpus == 64 and np.bincount(pl.owner).tolist() == [4] * 64
    T.save_topology(tmp_path / "t.json", topo, pl)
    t2, p2 = T.load_topology(tmp_path / "t.json")
    assert t2 == topo and np.array_equal(p2.owner, pl.owner)
    with pytest.raises(ValueError):
        T.ClusterTopology(0, 1)


# ---- the C-ABI library -------------------------------------------------------

HEADER = ROOT / "include" / "fusco.h"


def header_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fs_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2512_22036_b200 import _lib

    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _lib.SIGNATURES, f"{s} missing a ctypes signature"
    assert lib.fs_abi_version() == 2


def test_library_validates_before_touching_cuda(monkeypatch):
    """Argument errors come back as ValueError without needing a GPU."""
    from ctypes import byref, c_size_t, c_void_p

    from paper_2512_22036_b200 import _lib

    n = c_size_t()
    _lib.call("fs_region_bytes", 8, 256, 8, 14336, 300, 1000, 1, byref(n))
    # signal block + 2 parity copies of the epoch-tagged count words (u64 P x
    # (E + 1)) + the dispatch block words (u64 P x ceil(300 / 128)) + the
    # duplicate lists (int2 P x 300 x (K - 1)) + the activation rows + the
    # expert-output rows + the owner pre-reduction records (80 B P x 300)
    # and fp32 partials (P x 300 x 2 tb)
    a256 = lambda b: (b + 255) // 256 * 256  # noqa: E731
    fixed = 4096 + 2 * a256(8 * 257 * 8) + a256(8 * 3 * 8) + a256(8 * 300 * 7 * 8)
    reduce = a256(8 * 300 * 80) + 8 * 300 * 2 * 14336
    assert n.value == fixed + 2 * a256(1000 * 14336) + reduce
    _lib.call("fs_region_bytes", 8, 256, 8, 14336, 300, 1000, 0, byref(n))
    assert n.value == fixed + a256(1000 * 14336) + reduce
    monkeypatch.setenv("FUSCO_OWNER_REDUCE", "0")  # no pre-reduction buffers
    _lib.call("fs_region_bytes", 8, 256, 8, 14336, 300, 1000, 0, byref(n))
    assert n.value == fixed + a256(1000 * 14336)
    monkeypatch.delenv("FUSCO_OWNER_REDUCE")
    with pytest.raises(ValueError):
        _lib.call("fs_region_bytes", 0, 256, 8, 14336, 300, 1000, 1, byref(n))
    owner = (np.arange(8) % 2).astype(np.int32)
    peers = (c_void_p * 2)(1, 2)
    h = c_void_p()
    with pytest.raises(ValueError):  # topk > num_experts
        _lib.call("fs_create", 0, 0, 2, 8, 9, 64, 16, 0, 0, owner.ctypes.data_as(c_void_p), None, peers, 0, 0,
                  byref(h))
    with pytest.raises(ValueError):  # token_bytes not a multiple of 4
        _lib.call("fs_create", 0, 0, 2, 8, 2, 66, 16, 0, 0, owner.ctypes.data_as(c_void_p), None, peers, 0, 0,
                  byref(h))
    bad_owner = np.full(8, 5, dtype=np.int32)
    with pytest.raises(ValueError):  # owner outside [0, world)
        _lib.call("fs_create", 0, 0, 2, 8, 2, 64, 16, 0, 0, bad_owner.ctypes.data_as(c_void_p), None, peers, 0, 0,
                  byref(h))
    with pytest.raises(ValueError):
        _lib.call("fs_layout", None, None, 4, 0, None, None, None, None, None, None, 3, None)
    assert "null handle" in _lib.load().fs_last_error().decode()


def test_no_cpu_fallback_in_product_path():
    """The product package never imports the oracle (test infrastructure)."""
    pkg = ROOT / "paper_2512_22036_b200"
    for py in pkg.rglob("*.py"):
        src = py.read_text()
        assert "import oracle" not in src and "from oracle" not in src, py


def _matrix_cfg():
    from paper_2512_22036_b200 import matrix as M

    topo, pl = T.preset("test")
    return M, M.BenchConfig(topo, pl, ("realworld", "imbalanced"), (256, 512), topk=4, token_bytes=64, repeats=1)


def test_bench_matrix_cells_fingerprint_and_render():
    """Matrix structure mirrors the reference (bench.py:48-160): pattern-major
    cells, per-cell SeedSequence((seed, index)) routing, stable sha256
    fingerprint that changes with the config, JSON/CSV/MD emitters."""
    M, cfg = _matrix_cfg()
    assert M.cells(cfg) == [("realworld", 256), ("realworld", 512), ("imbalanced", 256), ("imbalanced", 512)]
    a1 = M.cell_assignment(cfg, 1, "realworld", 512)
    a2 = M.cell_assignment(cfg, 1, "realworld", 512)
    assert a1.num_tokens == 512 and np.array_equal(a1.experts, a2.experts)
    assert not np.array_equal(M.cell_assignment(cfg, 0, "realworld", 512).experts, a1.experts)
    fp = cfg.fingerprint()
    assert len(fp) == 64 and fp == M.BenchConfig(cfg.topo, cfg.placement, cfg.patterns, cfg.seq_lens, topk=4,
                                                 token_bytes=64, repeats=1).fingerprint()
    assert fp != M.BenchConfig(cfg.topo, cfg.placement, cfg.patterns, cfg.seq_lens, topk=4, token_bytes=128,
                               repeats=1).fingerprint()
    row = {k: 0 for k in M.ROW_FIELDS}
    row.update(pattern="realworld", seq_len=16, variant="fused", mode="gpu", balancer="greedy", dedup_ratio=1.5,
               total_s=1e-5, latency_us=10.0, routed_gbps=1.0)
    doc = {"schema": M.SCHEMA_ID, "fingerprint": fp, "config": cfg.fingerprint_doc(), "rows": [row]}
    M.validate_result(doc)
    assert M.render(doc, "csv").splitlines()[0].split(",") == list(M.ROW_FIELDS)
    assert "| realworld | 16 | fused |" in M.render(doc, "md")
    import json

    assert json.loads(M.render(doc, "json"))["rows"][0]["variant"] == "fused"
    with pytest.raises(ValueError):
        M.validate_result({**doc, "rows": [{**row, "variant": "nope"}]})
    with pytest.raises(ValueError):
        M.validate_result({**doc, "rows": [{k: v for k, v in row.items() if k != "dedup_ratio"}]})


def test_bench_matrix_trace_and_topology_file(tmp_path):
    """--trace / --topology FILE (reference bench.py:291-298, 343-346,
    374-383): a recorded routing replaces the generated cells, its label
    enters the fingerprint; a bad file is an argument error (exit code 2)."""
    import paper_2512_22036_b200 as pkg
    from paper_2512_22036_b200 import matrix as M

    topo, pl = pkg.preset("test")
    a = pkg.gen_realworld(300, 4, topo, pl, seed=3)
    tr = tmp_path / "captured.json"
    pkg.save_trace(tr, a, 96)
    topo_file = tmp_path / "topo.json"
    pkg.save_topology(topo_file, topo, pl)
    back, tb = pkg.load_trace(tr)
    cfg = M.BenchConfig(topo, pl, topk=4, token_bytes=tb, trace=back, trace_label=tr.name)
    assert M.cells(cfg) == [("captured.json", 300)]
    assert np.array_equal(M.cell_assignment(cfg, 0, "captured.json", 300).experts, a.experts)
    assert cfg.fingerprint_doc()["trace"] == "captured.json"
    assert cfg.fingerprint() != M.BenchConfig(topo, pl, topk=4, token_bytes=tb).fingerprint()
    assert M.main(["--topology", str(tmp_path / "missing.json")]) == 2
    bad = tmp_path / "bad.json"
    bad.write_text("{}")
    assert M.main(["--topology", str(topo_file), "--trace", str(bad)]) == 2


# ---- wire / golden formats (§8f #4) -----------------------------------------


def test_descriptor_wire_format():
    """descriptor.py:224-241: LE u64 count, then (offset, length) u64 pairs."""
    import struct

    from paper_2512_22036_b200 import wire as W

    blob = W.descriptor_to_bytes([8, 0], [4, 4])
    assert blob == struct.pack("<QQQQQ", 2, 8, 4, 0, 4)
    off, ln = W.descriptor_from_bytes(blob)
    assert off.tolist() == [8, 0] and ln.tolist() == [4, 4]
    assert W.descriptor_from_bytes(W.descriptor_to_bytes([], []))[0].size == 0
    with pytest.raises(ValueError):
        W.descriptor_from_bytes(b"\x01\x00")
    with pytest.raises(ValueError):
        W.descriptor_from_bytes(blob[:-1])
    with pytest.raises(ValueError):
        W.descriptor_to_bytes([1, 2], [3])
    ref = Path("/root/reference/pkg/src")
    if ref.is_dir():  # the reference's own encoder, when present in this container
        import sys

        sys.path.insert(0, str(ref))
        try:
            from shuffleforge.descriptor import DescriptorList
        finally:
            sys.path.remove(str(ref))
        d = DescriptorList("x", np.array([8, 0, 96]), np.array([4, 4, 32]))
        assert d.to_bytes() == W.descriptor_to_bytes([8, 0, 96], [4, 4, 32])


def _oracle_plans(g):
    """GpuPlan pair built from the oracle's layouts (what the device plan must equal)."""
    from oracle import shuffle_oracle as O
    from paper_2512_22036_b200.api import ActivationLayout, GpuPlan

    P = g["num_nodes"] * g["gpus_per_node"]
    lays, row_of = O.activation_layouts(g["experts"], g["source"], g["owner"], P)
    layouts = {r: ActivationLayout(l.expert_ids, l.token_ids, l.src, l.k_col) for r, l in lays.items()}
    local = {s: np.flatnonzero(g["source"] == s) for s in range(P)}
    tb, K, T = g["token_bytes"], g["topk"], g["experts"].shape[0]

    def mk(direction):
        return GpuPlan(direction=direction, token_bytes=tb, num_tokens=T, topk=K, groups=None, layouts=layouts,
                       local_tokens=local, row_of=row_of, first_mask=g["first_mask"], reduce_weights=None,
                       inter_bytes_total=0, intra_bytes_total=0, intra_gpu_bytes=0, buffer_bytes={},
                       loads=g["loads"])
    return mk("dispatch"), mk("combine"), lays, row_of


@pytest.mark.parametrize("name", golden_names())
def test_plan_json_executes_to_reference_bytes(name):
    """The dumped plan (reference plan_to_json schema) is executable: applying
    its descriptor tables moves exactly the reference's bytes — dispatch
    activations equal the golden ones, every row written once, each token sent
    once per destination rank; combine staging reduces to the golden outputs."""
    import base64

    from oracle import shuffle_oracle as O
    from paper_2512_22036_b200 import wire as W

    g = load_golden(name)
    tb, K, T = g["token_bytes"], g["topk"], g["experts"].shape[0]
    P = g["num_nodes"] * g["gpus_per_node"]
    dplan, cplan, lays, row_of = _oracle_plans(g)
    dj = W.plan_to_json(dplan, g["gpus_per_node"])
    # layouts: exactly the reference's (golden rows concatenated over ranks)
    for key, gk in (("expert_ids", "lay_expert_ids"), ("token_ids", "lay_token_ids"), ("k_col", "lay_k_col")):
        got = np.concatenate([np.asarray(dj["layouts"][str(r)][key], dtype=np.int64) for r in range(P)])
        assert np.array_equal(got, g[gk])
    tables = lambda d: W.descriptor_from_bytes(base64.b64decode(d["table"]))  # noqa: E731
    payload = O.encode(np.random.default_rng(0).standard_normal((T, tb // 4)).astype(np.float32), "f32")
    bufs = {f"token/{s}": payload[np.flatnonzero(g["source"] == s)].reshape(-1).copy() for s in range(P)}
    for r in range(P):
        bufs[f"activation/{r}"] = np.zeros(lays[r].num_rows * tb, dtype=np.uint8)
    written = {r: np.zeros(lays[r].num_rows, dtype=np.int64) for r in range(P)}
    sent = np.zeros((T, P), dtype=np.int64)

    def apply(item):
        so, sl = tables(item["send"])
        ro, rl = tables(item["recv"])
        assert (sl == tb).all() and (rl == tb).all() and so.size == ro.size
        src, dst = bufs[item["send"]["buffer"]], bufs[item["recv"]["buffer"]]
        for a, b in zip(so, ro):
            dst[b : b + tb] = src[a : a + tb]
        if item["recv"]["buffer"].startswith("activation/"):
            written[int(item["recv"]["buffer"].split("/")[1])][ro // tb] += 1
        return so

    for tr in dj["node_transfers"]:
        so = apply(tr)
        toks = np.flatnonzero(g["source"] == tr["src_flat"])[so // tb]
        sent[toks, tr["dst_flat"]] += 1
        assert tr["bytes"] == so.size * tb
    for nd in sorted(dj["local_edges"]):
        for e in dj["local_edges"][nd]:
            if e["send"]["buffer"].startswith("token/"):
                apply(e)
    for nd in sorted(dj["local_edges"]):  # receiver fan-out after the primaries landed
        for e in dj["local_edges"][nd]:
            if e["send"]["buffer"].startswith("activation/"):
                apply(e)
    acts = O.dispatch(payload, lays)
    for r in range(P):
        assert np.array_equal(bufs[f"activation/{r}"].reshape(-1, tb), acts[r])
        assert (written[r] == 1).all()
    own = g["owner"][g["experts"]]
    want_sent = np.zeros((T, P), dtype=np.int64)
    for t in range(T):
        for d in set(own[t].tolist()) - {int(g["source"][t])}:
            want_sent[t, d] = 1
    assert np.array_equal(sent, want_sent)  # once per (token, remote rank)

    cj = W.plan_to_json(cplan, g["gpus_per_node"])
    staging = {s: np.zeros(((g["source"] == s).sum() * K) * tb, dtype=np.uint8) for s in range(P)}
    act_out = {f"act_out/{r}": acts[r].reshape(-1) for r in range(P)}
    items = cj["node_transfers"] + [e for nd in cj["local_edges"] for e in cj["local_edges"][nd]]
    for it in items:
        so, _ = tables(it["send"])
        ro, _ = tables(it["recv"])
        src = act_out[it["send"]["buffer"]]
        dst = staging[int(it["recv"]["buffer"].split("/")[1])]
        for a, b in zip(so, ro):
            dst[b : b + tb] = src[a : a + tb]
    assert sum(it["bytes"] for it in items) == T * K * tb
    for s in range(P):
        ids = np.flatnonzero(g["source"] == s)
        stg = O.decode(staging[s].reshape(-1, tb), "f32").reshape(ids.size, K, -1).astype(np.float64)
        out = np.zeros((ids.size, tb // 4), dtype=np.float64)
        for k in range(K):
            out = out + g["weights"][ids, k : k + 1] * stg[:, k]
        want = O.combine(acts, row_of, g["experts"], g["weights"], g["owner"], ids, "f32")
        assert np.array_equal(O.encode(out.astype(np.float32), "f32"), want)


def test_header_constants_and_signatures_match_binding():
    """include/fusco.h is the contract: every FS_* constant the Python binding
    mirrors has the header's value, and every ctypes signature has the
    prototype's parameter count."""
    from paper_2512_22036_b200 import _lib

    text = HEADER.read_text()
    defines = dict(re.findall(r"#define\s+(FS_[A-Z0-9_]+)\s+\(?(-?\d+)\)?", text))
    checked = 0
    for name, val in vars(_lib).items():
        if name.startswith("FS_") and isinstance(val, int) and name in defines:
            assert val == int(defines[name]), name
            checked += 1
    assert checked >= 10
    body = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    for name, params in re.findall(r"\b(fs_[a-z0-9_]+)\s*\(([^)]*)\)\s*;", body, flags=re.S):
        n = 0 if params.strip() in ("", "void") else params.count(",") + 1
        assert len(_lib.SIGNATURES[name][1]) == n, name


@pytest.mark.parametrize("cfg,P,want", [
    ("mixtral", 2, (50.3, 50.7, 64.1, 64.4)),
    ("mixtral", 8, (112.0, 113.2, 112.0, 113.2)),
    ("qwen3", 8, (74.9, 75.2, 112.1, 113.1)),
    ("dsv3", 8, (259.2, 261.8, 391.7, 396.4)),
    ("dsv3_decode", 8, (8.1, 8.5, 12.3, 13.0)),
    ("dsv3_zipf", 4, (154.7, 167.5, 336.0, 484.7)),
])
def test_bench_traffic_matches_reference_volumes(cfg, P, want):
    """The NVLink byte accounting behind every multi-GPU roofline (bench.traffic)
    reproduces SURVEY.md §8d's table, computed from the reference's own plans
    (MiB: dispatch mean egress, dispatch max(eg, in), combine mean egress,
    combine max(eg, in)); the dispatch egress equals dispatch_loads."""
    import bench
    from oracle import shuffle_oracle as O

    hidden, dtype, E, K, T_l, _, _ = bench.CONFIGS[cfg]
    a, pl = bench.routing_for(cfg, P, 0)
    tb = hidden * (2 if dtype == "bf16" else 4)
    tr = bench.traffic(a.experts, a.source, pl.owner, P, tb, T_l)
    M = 2**20
    got = (tr["d_eg"].mean() / M, np.maximum(tr["d_eg"], tr["d_in"]).max() / M,
           tr["c_eg"].mean() / M, np.maximum(tr["c_eg"], tr["c_in"]).max() / M)
    assert np.allclose(got, want, atol=0.051), got
    assert np.array_equal(tr["d_eg"], O.dispatch_loads(a.experts, a.source, pl.owner, P, tb, 1))


@pytest.mark.parametrize("cfg,P", [("dsv3", 2), ("dsv3_zipf", 4), ("qwen3", 2), ("dsv3_decode", 2)])
def test_bench_traffic_owner_reduced_bytes(cfg, P):
    """The combine bytes with owner-side pre-reduction (bench.traffic's
    c_eg_red / c_in_red, the figure ncu's NVLink counters matched): per
    (token, remote owner) group of m rows, one fp32 partial (2 tb) when
    m >= 3, else the m rows -- brute force over the routing."""
    import bench

    hidden, dtype, E, K, T_l, _, _ = bench.CONFIGS[cfg]
    a, pl = bench.routing_for(cfg, P, 0)
    tb = hidden * 2
    tr = bench.traffic(a.experts, a.source, pl.owner, P, tb, T_l)
    own = pl.owner[a.experts]
    eg = np.zeros(P)
    ing = np.zeros(P)
    for t in range(a.num_tokens):
        s = a.source[t]
        for g in range(P):
            m = int((own[t] == g).sum())
            if g == s or m == 0:
                continue
            b = 2 * tb if m >= 3 else m * tb
            eg[g] += b
            ing[s] += b
    assert np.array_equal(tr["c_eg_red"], eg) and np.array_equal(tr["c_in_red"], ing)
    assert (tr["c_eg_red"] <= tr["c_eg"]).all()
