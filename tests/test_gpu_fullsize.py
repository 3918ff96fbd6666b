"""Parity at the BASELINE.json sizes, on one B200 with the P ranks emulated
(every kernel addresses its "peers" through the same pointer table it uses
over NVLink; regions of up to 3.8 GB per rank).

Two kinds of evidence:

* **Reference digests.**  ``tests/golden/digests.json`` holds sha256 digests
  of the reference's own activation bytes, output bytes and ``row_of``,
  written by ``tests/golden/make_digests.py`` from ``shuffleforge.run_exchange``
  in the build container (oracle config 2 x 4096 tokens fp32, DeepSeek-V3
  decode EP=8, Qwen3 EP=8 and Mixtral EP=2 at full size, DeepSeek-V3 Zipf
  EP=4).  The CUDA path, fed the same routing and payloads, must hash
  identically: activations and layout bit-exact, outputs bit-exact with the
  f64 k-ascending reduction.
* **Oracle at full size (bf16).**  DeepSeek-V3 (uniform and Zipf s=1.2),
  Qwen3, Mixtral EP=2/4/8 and the single-GPU DeepSeek-V3 Zipf case:
  ``row_of``, per-expert counts/offsets, first_mask, rank mask and the dedup
  counters equal the oracle's (``planner.py:138-196``) exactly; every
  activation row equals its token's row (the oracle's dispatch, evaluated on
  the device); f64-accumulate outputs equal the oracle's reduction bit for
  bit on 1024 sampled tokens per source rank; the production fp32-accumulate
  outputs are within the bf16 tolerance of the f64 reduction for every
  token.  These exercise the multi-chunk planner with E=256, K=8 at P>1,
  which the smaller parity cases never reach.
"""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import shuffle_oracle as O
from test_gpu_parity import BF16_TOL, _check_layout

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

DIGESTS = json.loads((Path(__file__).resolve().parent / "golden" / "digests.json").read_text())


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2512_22036_b200 import _lib

    _lib.load()
    torch.cuda.set_device(0)
    yield
    torch.cuda.empty_cache()


def _pkg():
    import paper_2512_22036_b200 as pkg

    return pkg


def _sha(t) -> str:
    a = t.contiguous().view(torch.uint8).cpu().numpy() if isinstance(t, torch.Tensor) else np.ascontiguousarray(t)
    return hashlib.sha256(a.view(np.uint8).reshape(-1).data).hexdigest()


# ---------------------------------------------------------------------------
# pinned to the reference itself


@pytest.mark.parametrize("name", sorted(DIGESTS))
def test_full_size_matches_reference_digests(name):
    from paper_2512_22036_b200.engine import EmulatedCluster

    pkg = _pkg()
    d = DIGESTS[name]
    P, E, K, T_l, tb = d["P"], d["experts"], d["topk"], d["tokens_per_rank"], d["token_bytes"]
    topo = pkg.box(P)
    pl = pkg.round_robin_placement(E, topo)
    a = pkg.gen_realworld(P * T_l, K, topo, pl, seed=d["seed"], zipf_s=d["zipf_s"])
    payload = pkg.make_token_payloads(a.num_tokens, tb, d["payload_seed"])
    ids = [np.flatnonzero(a.source == s) for s in range(P)]
    with EmulatedCluster(P, E, K, tb, max(i.size for i in ids), owner=pl.owner) as cl:
        dev = cl.device
        idx = [torch.as_tensor(a.experts[i], device=dev) for i in ids]
        xs = [torch.as_tensor(payload[i], device=dev) for i in ids]
        ws = [torch.as_tensor(a.weights[i], dtype=torch.float64, device=dev) for i in ids]
        plans = cl.layout(idx, with_masks=False)
        cl.dispatch(xs, plans)
        outs = [torch.empty((i.size, tb // 4), dtype=torch.float32, device=dev) for i in ids]
        cl.combine(plans, ws, outs, dtype_code=0, acc=1)  # f32 payload, f64 accumulate
        cl.check()
        row_of = np.empty((a.num_tokens, K), dtype=np.int64)
        for s, p in enumerate(plans):
            row_of[ids[s]] = p.row_of.cpu().numpy()
        assert _sha(row_of) == d["row_of"], "row_of differs from the reference"
        for g in range(P):
            rows = plans[g].num_rows
            assert rows == d["act_rows"][g]
            assert _sha(cl.ranks[g].act(rows)) == d["activation"][g], f"activation/{g}"
        for s in range(P):
            assert _sha(outs[s]) == d["output"][s], f"output/{s} (f64 accumulate) differs from the reference"
        loads = [int(p.stats[4].item()) * tb for p in plans]
        assert loads == d["loads"]


# ---------------------------------------------------------------------------
# bf16 at the BASELINE sizes against the oracle


FULL = [
    # P, E, K, T_l, hidden, zipf, expert (expert "scaled+reduce": owner pre-reduction forced on)
    pytest.param(8, 256, 8, 4096, 7168, 0.0, "scaled", id="dsv3-ep8"),
    pytest.param(8, 256, 8, 4096, 7168, 1.2, "scaled+reduce", id="dsv3-zipf-ep8-reduce"),
    pytest.param(2, 256, 8, 4096, 7168, 0.0, "scaled", id="dsv3-ep2"),          # pre-reduction by default
    pytest.param(4, 256, 8, 4096, 7168, 1.2, "identity", id="dsv3-zipf-ep4"),   # pre-reduction by default
    pytest.param(8, 256, 8, 4096, 7168, 1.2, "identity", id="dsv3-zipf-ep8"),
    pytest.param(1, 256, 8, 4096, 7168, 1.2, "identity", id="dsv3-zipf-p1"),
    pytest.param(8, 256, 8, 128, 7168, 0.0, "scaled", id="dsv3-decode-ep8"),
    pytest.param(8, 128, 8, 4096, 2048, 0.0, "scaled", id="qwen3-ep8"),
    pytest.param(2, 8, 2, 8192, 4096, 0.0, "identity", id="mixtral-ep2"),
    pytest.param(4, 8, 2, 8192, 4096, 0.0, "scaled", id="mixtral-ep4"),
    pytest.param(8, 8, 2, 8192, 4096, 0.0, "identity", id="mixtral-ep8"),
]


def _scaled_gpu(act_bf16: torch.Tensor, e: torch.Tensor) -> torch.Tensor:
    """The reference scaled_expert (engine.py:283-292) in f32, rounded to bf16
    (same operation order as oracle.scaled_expert + encode)."""
    ef = e.to(torch.float32)[:, None]
    return (act_bf16.float() * (ef + 2) + ef).to(torch.bfloat16)


@pytest.mark.parametrize("P,E,K,T_l,hidden,zipf,expert", FULL)
def test_full_size_bf16_against_oracle(monkeypatch, P, E, K, T_l, hidden, zipf, expert):
    from paper_2512_22036_b200.engine import EmulatedCluster

    if expert.endswith("+reduce"):
        monkeypatch.setenv("FUSCO_OWNER_REDUCE", "1")
        expert = expert.split("+")[0]

    pkg = _pkg()
    topo = pkg.box(P)
    pl = pkg.round_robin_placement(E, topo)
    a = pkg.gen_realworld(P * T_l, K, topo, pl, seed=P * 11 + K, zipf_s=zipf)
    tb = hidden * 2
    ids = [np.flatnonzero(a.source == s) for s in range(P)]
    scaled = expert == "scaled"
    with EmulatedCluster(P, E, K, tb, T_l, owner=pl.owner, with_act_out=scaled) as cl:
        dev = cl.device
        gen = torch.Generator(device=dev).manual_seed(P * 1000 + E)
        x_all = torch.randn(a.num_tokens, hidden, generator=gen, device=dev).to(torch.bfloat16)
        idx = [torch.as_tensor(a.experts[i], device=dev) for i in ids]
        xs = [x_all[torch.as_tensor(i, device=dev)].contiguous() for i in ids]
        src = 1 if scaled else 0

        def run(acc):
            plans = cl.layout(idx)
            wdt = torch.float64 if acc == "f64" else torch.float32
            ws = [torch.as_tensor(a.weights[i], dtype=wdt, device=dev) for i in ids]
            # the router weights reach the dispatch (owner pre-reduction for the
            # fp32 combine where the library enables it; never for f64)
            cl.dispatch(xs, plans, ws=ws)
            if scaled:
                for r, p in zip(cl.ranks, plans):
                    n = p.num_rows
                    e = torch.repeat_interleave(torch.as_tensor(r.local_experts, device=dev),
                                                p.expert_counts.to(torch.int64))
                    r.act_out(n, torch.bfloat16).copy_(_scaled_gpu(r.act(n, torch.bfloat16), e))
            outs = [torch.empty((i.size, hidden), dtype=torch.bfloat16, device=dev) for i in ids]
            cl.combine(plans, ws, outs, dtype_code=1, src=src, acc=1 if acc == "f64" else 0)
            cl.check()
            return plans, outs

        plans, out64 = run("f64")
        res = dict(row_of=[p.row_of.cpu().numpy() for p in plans],
                   counts=[p.expert_counts.cpu().numpy() for p in plans],
                   offsets=[p.expert_offsets.cpu().numpy() for p in plans],
                   stats=[p.stats.cpu().numpy() for p in plans],
                   first=[p.first_mask.cpu().numpy() for p in plans],
                   rank_mask=[p.rank_mask.cpu().numpy() for p in plans], ids=ids)
        layouts, row_of = _check_layout(res, a, pl, P)
        x_u8 = x_all.view(torch.uint8).reshape(a.num_tokens, tb)
        for g in range(P):
            rows = layouts[g].num_rows
            want = O.dispatch(x_u8, {g: layouts[g]})[g] if rows else x_u8[:0]
            assert torch.equal(cl.ranks[g].act(rows), want), f"activation/{g}"
        # f64-accumulate combine: bit-exact with the oracle's reduction on sampled tokens
        rng = np.random.default_rng(P + K)
        x_host = {}
        for s in range(P):
            n = ids[s].size
            loc = np.sort(rng.choice(n, size=min(n, 1024), replace=False))
            t = ids[s][loc]
            xh = x_u8[torch.as_tensor(t, device=dev)].cpu().numpy()
            x_host[s] = (loc, t, xh)

            def rows_of(k, t=t, xh=xh):
                if not scaled:
                    return xh
                return O.encode(O.scaled_expert(O.decode(xh, "bf16"), a.experts[t, k]), "bf16")

            want = O.reduce_rows(rows_of, a.weights[t], "bf16")
            got = out64[s].view(torch.uint8)[torch.as_tensor(loc, device=dev)].cpu().numpy()
            assert np.array_equal(got, want), f"output/{s}: f64-accumulate combine not bit-exact"
        # production fp32-accumulate combine, every token, against the f64 reduction
        _, out32 = run("f32")
        for s in range(P):
            w = torch.as_tensor(a.weights[ids[s]], dtype=torch.float64, device=dev)
            acc = torch.zeros((ids[s].size, hidden), dtype=torch.float64, device=dev)
            for k in range(K):
                y = xs[s]
                if scaled:
                    y = _scaled_gpu(y, torch.as_tensor(a.experts[ids[s], k], device=dev))
                acc = acc + w[:, k : k + 1] * y.double()
            torch.testing.assert_close(out32[s].double(), acc, **BF16_TOL)
