"""The reference's executor API on the GPU path: build_plan_pair /
build_dispatch_plan / build_combine_plan, allocate_buffers,
fill_token_buffers, apply_node_level, apply_expert_level, run_experts,
reduce_outputs (reference engine.py:249-338, planner.py:211-497) and SPEC's
execute_dispatch / execute_combine, driven exactly as the
reference's run_exchange drives them (engine.py:429-437) on the reference's
own round-trip cases (test_engine.py:185-205): activations bit-exact,
outputs bit-exact (f64 k-ascending reduction)."""

import numpy as np
import pytest

from oracle import shuffle_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2512_22036_b200 import _lib

    _lib.load()
    torch.cuda.set_device(0)


def _small_case(seed=0, num_tokens=96, topk=4, tb=64):
    """reference test_engine.py:27-30 small_case (preset "test")."""
    import paper_2512_22036_b200 as pkg

    topo, placement = pkg.preset("test")
    a = pkg.gen_realworld(num_tokens, topk, topo, placement, seed=seed)
    return pkg, topo, placement, a, tb


def _oracle(a, placement, topo, payloads, expert):
    fn = O.scaled_expert if expert == "scaled" else O.identity_expert
    return O.exchange(a.experts, a.weights, a.source, placement.owner, topo.num_gpus, payloads, fn, "f32",
                      topo.gpus_per_node)


def _host(t):
    return t.cpu().numpy()


@pytest.mark.parametrize("seed,payload_seed,expert", [(3, 11, "identity"), (4, 7, "scaled"), (9, 2, "scaled")])
def test_executor_stages_match_reference_round_trip(seed, payload_seed, expert):
    pkg, topo, pl, a, tb = _small_case(seed=seed)
    d, c, groups = pkg.build_plan_pair(a, topo, pl, tb)
    bufs = pkg.allocate_buffers(d, c)
    payloads = pkg.make_token_payloads(a.num_tokens, tb, payload_seed)
    pkg.fill_token_buffers(d, bufs, payloads)
    fn = pkg.scaled_expert(pl.num_experts) if expert == "scaled" else pkg.identity_expert
    pkg.apply_node_level(d, bufs)
    pkg.apply_expert_level(d, bufs)
    pkg.run_experts(c, bufs, fn)
    pkg.apply_expert_level(c, bufs)
    pkg.apply_node_level(c, bufs)
    pkg.reduce_outputs(c, bufs)
    want = _oracle(a, pl, topo, payloads, expert)
    for g in range(topo.num_gpus):
        lay = d.layouts[g]
        act = _host(bufs[f"activation/{g}"]).reshape(lay.num_rows, tb)
        assert np.array_equal(act, payloads[lay.token_ids]), f"activation/{g}"
        assert d.buffer_bytes[f"activation/{g}"] == bufs[f"activation/{g}"].numel()
    for s in range(topo.num_gpus):
        assert np.array_equal(_host(bufs[f"output/{s}"]), want["outputs"][s].reshape(-1)), f"output/{s}"


def test_spec_execute_dispatch_and_combine():
    pkg, topo, pl, a, tb = _small_case(seed=5, num_tokens=200, topk=4, tb=128)
    d, c, _ = pkg.build_plan_pair(a, topo, pl, tb)
    bufs = pkg.allocate_buffers(d, c)
    payloads = pkg.make_token_payloads(a.num_tokens, tb, 3)
    pkg.fill_token_buffers(d, bufs, payloads)
    acts, drep = pkg.execute_dispatch(d, bufs)
    assert drep.direction == "dispatch" and drep.rearrange_bytes == 0 and drep.communicate_s > 0
    assert drep.inter_node_bytes == d.inter_bytes_total
    pkg.run_experts(c, bufs, pkg.scaled_expert(pl.num_experts))
    outs, crep = pkg.execute_combine(c, bufs, a.weights)
    assert crep.direction == "combine" and crep.rearrange_bytes == 0
    want = _oracle(a, pl, topo, payloads, "scaled")
    for g in range(topo.num_gpus):
        assert np.array_equal(_host(acts[g]).reshape(-1, tb), want["activations"][g])
    for s in range(topo.num_gpus):
        assert np.array_equal(_host(outs[s]), want["outputs"][s].reshape(-1))
    # a second combine of the same plan with other weights (uniform 1/K)
    w2 = np.full_like(a.weights, 1.0 / a.topk)
    outs2, _ = pkg.execute_combine(c, bufs, w2)
    want2 = O.exchange(a.experts, w2, a.source, pl.owner, topo.num_gpus, payloads, O.scaled_expert, "f32")
    for s in range(topo.num_gpus):
        assert np.array_equal(_host(outs2[s]), want2["outputs"][s].reshape(-1))


def test_repeated_dispatch_and_separately_built_plans():
    pkg, topo, pl, a, tb = _small_case(seed=6, num_tokens=150)
    groups = pkg.static_groups(topo)
    d = pkg.build_dispatch_plan(a, topo, pl, tb, groups)
    c = pkg.build_combine_plan(a, topo, pl, tb, groups)
    dp, _, _ = pkg.build_plan_pair(a, topo, pl, tb)
    for g in range(topo.num_gpus):
        assert np.array_equal(d.layouts[g].token_ids, dp.layouts[g].token_ids)
    assert d.inter_bytes_total == dp.inter_bytes_total  # groups change forwarders, not volume
    bufs = pkg.allocate_buffers(d, c)
    want = None
    for it in range(3):  # the same plan executed three times (each a new device epoch)
        payloads = pkg.make_token_payloads(a.num_tokens, tb, 20 + it)
        pkg.fill_token_buffers(d, bufs, payloads)
        pkg.execute_dispatch(d, bufs)
        pkg.execute_combine(c, bufs)
        want = _oracle(a, pl, topo, payloads, "identity")
        for g in range(topo.num_gpus):
            assert np.array_equal(_host(bufs[f"activation/{g}"]).reshape(-1, tb), want["activations"][g])
            assert np.array_equal(_host(bufs[f"output/{g}"]), want["outputs"][g].reshape(-1))


def test_direct_plans_same_bytes_more_traffic():
    pkg, topo, pl, a, tb = _small_case(seed=7, num_tokens=120)
    d, c = pkg.build_direct_plans(a, topo, pl, tb)
    assert d.inter_bytes_total == pkg.naive_inter_node_bytes(a, pl, topo, tb)
    bufs = pkg.allocate_buffers(d, c)
    payloads = pkg.make_token_payloads(a.num_tokens, tb, 1)
    pkg.fill_token_buffers(d, bufs, payloads)
    pkg.execute_dispatch(d, bufs)
    pkg.execute_combine(c, bufs)
    want = _oracle(a, pl, topo, payloads, "identity")
    for g in range(topo.num_gpus):
        assert np.array_equal(_host(bufs[f"activation/{g}"]).reshape(-1, tb), want["activations"][g])
        assert np.array_equal(_host(bufs[f"output/{g}"]), want["outputs"][g].reshape(-1))


def test_executor_errors_are_value_errors():
    pkg, topo, pl, a, tb = _small_case(seed=8, num_tokens=64)
    d, c, _ = pkg.build_plan_pair(a, topo, pl, tb)
    bufs = pkg.allocate_buffers(d, c)
    with pytest.raises(ValueError):
        pkg.apply_expert_level(d, bufs)  # expert level before node level
    with pytest.raises(ValueError):
        pkg.reduce_outputs(c, bufs)  # combine before dispatch
    with pytest.raises(ValueError):
        pkg.reduce_outputs(d, bufs)  # not a combine plan
    bad = dict(bufs)
    bad["activation/0"] = torch.zeros_like(bufs["activation/0"])  # not the symmetric rows
    with pytest.raises(ValueError):
        pkg.apply_node_level(d, bad)
    short = dict(bufs)
    short["token/1"] = bufs["token/1"][:-4]
    with pytest.raises(ValueError):
        pkg.apply_node_level(d, short)
    _, _, a2, _ = _small_case(seed=9, num_tokens=64)[1:]
    d2, _, _ = pkg.build_plan_pair(a2, topo, pl, tb)
    with pytest.raises(ValueError):
        pkg.allocate_buffers(d, d2)
    # still usable after the rejected calls
    payloads = pkg.make_token_payloads(a.num_tokens, tb, 0)
    pkg.fill_token_buffers(d, bufs, payloads)
    pkg.execute_dispatch(d, bufs)
    outs, _ = pkg.execute_combine(c, bufs)
    want = _oracle(a, pl, topo, payloads, "identity")
    for s in range(topo.num_gpus):
        assert np.array_equal(_host(outs[s]), want["outputs"][s].reshape(-1))
