"""Achievable NVLink / HBM bandwidth of the engines' own data movers.

    torchrun --nproc-per-node N tools/p2p_probe.py [MiB per pair]

Every rank allocates a symmetric region, maps every peer's (CUDA IPC), and
times with CUDA events (max over ranks):
  hbm    local copy src->dst (read+write bytes counted)
  push   all-to-all: each rank writes its slice to every peer   (egress/GPU)
  pull   all-to-all: each rank reads its slice from every peer  (ingress/GPU)
for mode warp (16 B LDG/STG) and tma (cp.async.bulk through smem).
Prints one JSON line (rank 0); bench.py uses the push/pull figures as the
in-run NVLink peak when a profile of this run is committed.
"""
import ctypes
import json
import os
import sys
from ctypes import byref, c_void_p
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2512_22036_b200 import _lib  # noqa: E402
from paper_2512_22036_b200.engine import exchange_objects  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    world = int(os.environ.get("WORLD_SIZE", 1))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank = dist.get_rank() if world > 1 else 0
    mib = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    per = mib << 20
    total = 2 * per * max(world, 1) + (1 << 20)
    own = c_void_p()
    _lib.call("fs_sym_alloc", local, total, byref(own))
    h = (ctypes.c_uint8 * 64)()
    _lib.call("fs_ipc_handle", local, own, h)
    infos = exchange_objects(bytes(h), None) if world > 1 else [bytes(h)]
    bases = []
    for g, hb in enumerate(infos):
        if g == rank:
            bases.append(own.value)
            continue
        p = c_void_p()
        _lib.call("fs_ipc_open", local, (ctypes.c_uint8 * 64).from_buffer_copy(hb), byref(p))
        bases.append(p.value)
    # region layout: [send slices: world x per][recv slices: world x per]
    send = lambda g, j: bases[g] + j * per  # noqa: E731
    recv = lambda g, j: bases[g] + (world + j) * per  # noqa: E731
    stream = _lib.stream_ptr()
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    res = {}
    sweep = os.environ.get("PROBE_SWEEP")  # e.g. "1,2,4,8": warp-mode CTAs per SM to try
    modes = [(0, f"warp{m}", sms * int(m)) for m in sweep.split(",")] if sweep else \
        [(0, "warp", sms * 4), (1, "tma", sms * 8)]
    for mode, name, ctas in modes:
        cases = {
            "hbm": ([recv(rank, 0)], [send(rank, 0)], 2),
            "push": ([recv(g, rank) for g in range(world) if g != rank],
                     [send(rank, g) for g in range(world) if g != rank], 1),
            "pull": ([recv(rank, g) for g in range(world) if g != rank],
                     [send(g, rank) for g in range(world) if g != rank], 1),
        }
        for cname, (dsts, srcs, factor) in cases.items():
            if not dsts:
                continue
            D = (c_void_p * len(dsts))(*dsts)
            S = (c_void_p * len(srcs))(*srcs)
            for _ in range(3):
                _lib.call("fs_probe_a2a", local, D, S, len(dsts), per, mode, ctas, stream)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 10
            e0.record()
            for _ in range(reps):
                _lib.call("fs_probe_a2a", local, D, S, len(dsts), per, mode, ctas, stream)
            e1.record()
            torch.cuda.synchronize()
            ms = torch.tensor([e0.elapsed_time(e1) / reps], device="cuda")
            if world > 1:
                dist.all_reduce(ms, op=dist.ReduceOp.MAX)
            gbs = factor * len(dsts) * per / (ms.item() * 1e-3) / 1e9
            res[f"{name}_{cname}_gbs"] = round(gbs, 1)
    if world > 1 and os.environ.get("PROBE_MIXED") == "1":
        # half of every pair's bytes pushed by the source, half pulled by the
        # destination, concurrently on two streams: same link direction
        half = per // 2
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        pd = [recv(g, rank) for g in range(world) if g != rank]
        ps = [send(rank, g) for g in range(world) if g != rank]
        ld = [recv(rank, g) + half for g in range(world) if g != rank]
        ls = [send(g, rank) + half for g in range(world) if g != rank]
        PD, PS = (c_void_p * len(pd))(*pd), (c_void_p * len(ps))(*ps)
        LD, LS = (c_void_p * len(ld))(*ld), (c_void_p * len(ls))(*ls)
        for mode, name in ((0, "warp"), (1, "tma")):
            ctas = sms * (2 if mode == 0 else 4)

            def go():
                _lib.call("fs_probe_a2a", local, PD, PS, len(pd), half, mode, ctas, c_void_p(s1.cuda_stream))
                _lib.call("fs_probe_a2a", local, LD, LS, len(ld), half, mode, ctas, c_void_p(s2.cuda_stream))
            for _ in range(3):
                go()
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 10
            cur = torch.cuda.current_stream()
            e0.record(cur)
            s1.wait_stream(cur)
            s2.wait_stream(cur)
            for _ in range(reps):
                go()
            cur.wait_stream(s1)
            cur.wait_stream(s2)
            e1.record(cur)
            torch.cuda.synchronize()
            ms = torch.tensor([e0.elapsed_time(e1) / reps], device="cuda")
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
            res[f"{name}_mixed_gbs"] = round(len(pd) * per / (ms.item() * 1e-3) / 1e9, 1)
    if rank == 0:
        print(json.dumps({"world": world, "mib_per_pair": mib, **res}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
