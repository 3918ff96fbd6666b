"""Multi-process host logic on CPU (gloo, world_size 2): the bootstrap that
precedes every multi-GPU shuffle, per-rank routing slices, and the bench's
per-rank traffic accounting — no GPU needed."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import shuffle_oracle as O


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, mode, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_22036_b200 import box, gen_realworld, local_routing, round_robin_placement
        from paper_2512_22036_b200.engine import bootstrap_exchange

        handle = bytes([rank]) * 64
        cfg = (world, 64, 8, 4096, 128, 0, True, tuple(range(8)), 0)
        if mode == "mismatch" and rank == 1:
            cfg = (world, 64, 8, 2048, 128, 0, True, tuple(range(8)), 0)
        try:
            hs = bootstrap_exchange(handle, cfg, rank)
            res = ("ok", [h[0] for h in hs])
        except ValueError as exc:
            res = ("error", str(exc))
        # every rank slices the same global routing identically
        topo = box(world)
        pl = round_robin_placement(16, topo)
        a = gen_realworld(world * 50, 4, topo, pl, seed=3)
        ids, idx, w = local_routing(a, rank)
        t = torch.tensor([float(idx.sum()), float(ids.size)])
        dist.all_reduce(t)
        # max-over-ranks timing reduction used by bench.py
        mx = torch.tensor([float(rank + 1)])
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        q.put((rank, res, t.tolist(), float(a.experts.sum()), mx.item()))
    finally:
        dist.destroy_process_group()


def _run(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out)


def test_bootstrap_agrees_and_orders_handles():
    out = _run("ok")
    for rank, res, tot, full_sum, mx in out:
        assert res == ("ok", [0, 1])
        assert tot[0] == full_sum and tot[1] == 100  # slices partition the global routing
        assert mx == 2.0


def test_bootstrap_rejects_mismatched_configuration():
    out = _run("mismatch")
    for rank, res, *_ in out:
        assert res[0] == "error" and "differs" in res[1]


def test_bench_traffic_accounting_matches_oracle():
    """bench.traffic (NVLink / HBM bytes per rank) against oracle counts."""
    import bench
    from paper_2512_22036_b200 import box, gen_realworld, round_robin_placement

    for P, E, K in ((2, 8, 2), (4, 32, 4), (8, 256, 8)):
        topo = box(P)
        pl = round_robin_placement(E, topo)
        a = gen_realworld(P * 64, K, topo, pl, seed=P)
        tb = 32
        tr = bench.traffic(a.experts, a.source, pl.owner, P, tb, 64)
        assert np.array_equal(tr["d_eg"].astype(np.int64), O.dispatch_loads(a.experts, a.source, pl.owner, P, tb))
        own = pl.owner[a.experts]
        remote = own != a.source[:, None]
        layouts, _ = O.activation_layouts(a.experts, a.source, pl.owner, P)
        assert np.array_equal(tr["rows"], [layouts[g].num_rows for g in range(P)])
        assert tr["c_in"].sum() == remote.sum() * tb == tr["c_eg"].sum()
        assert tr["d_in"].sum() == tr["d_eg"].sum()
        # every received row written once; duplicates of remote tokens read once more
        assert np.all(tr["hbm_disp"] >= 64 * tb + tr["rows"] * tb)
