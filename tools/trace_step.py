"""Per-phase device timeline of one shuffle step (globaltimer stamps, CTA 0).

    FUSCO_TRACE=1 python tools/trace_step.py [config] [warp|tma] [warp|tma]
    torchrun --nproc-per-node N tools/trace_step.py ...   (one timeline per rank)
"""
import ctypes
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ["FUSCO_TRACE"] = "1"
cfg = sys.argv[1] if len(sys.argv) > 1 else "mixtral"
os.environ["FUSCO_DISPATCH"] = sys.argv[2] if len(sys.argv) > 2 else "warp"
os.environ["FUSCO_COMBINE"] = sys.argv[3] if len(sys.argv) > 3 else os.environ["FUSCO_DISPATCH"]

import bench  # noqa: E402
from paper_2512_22036_b200 import EPBuffer, _lib  # noqa: E402

import torch.distributed as dist  # noqa: E402

hidden, dtype, E, K, T_l, zipf, desc = bench.CONFIGS[cfg]
world = int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
dev = torch.device("cuda", local)
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("nccl", device_id=dev)
rank = dist.get_rank() if world > 1 else 0
a, pl = bench.routing_for(cfg, world, 0)
sel = np.flatnonzero(a.source == rank)
buf = EPBuffer(num_experts=E, topk=K, hidden=hidden, dtype=dtype, max_tokens=T_l, with_act_out=False)
tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
x = torch.randn(T_l, hidden, device=dev).to(tdt)
idx = torch.as_tensor(a.experts[sel], device=dev)
w = torch.as_tensor(a.weights[sel], dtype=torch.float32, device=dev)
names = {0: "layout.begin", 6: "layout.staged", 7: "dispatch.signal", 1: "layout.hist", 15: "layout.totals", 2: "layout.gridsync", 3: "layout.publish", 4: "layout.wait",
         5: "layout.end", 8: "dispatch.begin", 9: "dispatch.pushed", 10: "dispatch.arrived", 11: "dispatch.end",
         12: "combine.begin", 13: "combine.ready", 14: "combine.end", 16: "layout.last_cta_exit", 19: "layout.scanned", 23: "layout.pre",
         17: "dispatch.last_cta_exit", 18: "combine.last_cta_exit"}
lib = _lib.load()
for it in range(30):
    plan = buf.build_plan(idx)
    buf.dispatch(x, plan)
    out = buf.combine(plan, w, src="act")
torch.cuda.synchronize()
if os.environ.get("TRACE_GRAPH") == "1":  # replay steps as one CUDA graph: no host gaps between kernels
    from paper_2512_22036_b200._lib import FS_PHASE_ALL, FS_SRC_ACT

    h = buf.r.handle
    P_ = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    side = torch.cuda.Stream()
    st = ctypes.c_void_p(side.cuda_stream)
    lay = (h, P_(idx), idx.element_size(), idx.shape[0], P_(plan.row_of), P_(plan.expert_counts),
           P_(plan.expert_offsets), None, None, P_(plan.stats), FS_PHASE_ALL, st)
    disp = (h, P_(x), P_(idx), idx.element_size(), P_(plan.row_of), idx.shape[0], FS_PHASE_ALL, st)
    comb = (h, P_(idx), idx.element_size(), P_(plan.row_of), P_(w), 4, idx.shape[0], P_(out), buf.dtype_code,
            FS_SRC_ACT, 0, FS_PHASE_ALL, st)
    side.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            for _ in range(4):
                lib.fs_layout(*lay)
                lib.fs_dispatch(*disp)
                lib.fs_combine(*comb)
    torch.cuda.current_stream().wait_stream(side)
    for _ in range(5):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        g.replay()
    torch.cuda.synchronize()
    buf.check()
tr = (ctypes.c_uint64 * 24)()
_lib.call("fs_trace", buf.r.handle, tr, _lib.stream_ptr())
t = np.array(list(tr), dtype=np.int64)
lines = [f"[rank {rank}] {cfg} world={world}"]
t0 = t[0]
if world > 1:  # common time origin: min layout.begin over ranks (globaltimer is per GPU; close enough)
    tt = torch.tensor([t0], dtype=torch.int64, device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MIN)
    t0 = int(tt.item())
prev = t0
for k in sorted(names, key=lambda k: t[k] if t[k] else 1 << 62):
    if t[k]:
        lines.append(f"  {names[k]:18s} {(t[k] - t0) / 1e3:9.2f} us  (+{(t[k] - prev) / 1e3:7.2f})")
        prev = t[k]
if world > 1:
    out = [None] * world
    dist.all_gather_object(out, "\n".join(lines))
    if rank == 0:
        print("\n".join(out), flush=True)
    dist.barrier()
    buf.close()
    dist.destroy_process_group()
else:
    print("\n".join(lines))
    buf.close()
