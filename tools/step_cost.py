"""Marginal cost of each kernel inside a graph-replayed single-GPU step.

    python tools/step_cost.py [config ...]

Captures CUDA graphs of (layout+dispatch+combine), (dispatch+combine),
(layout only), (dispatch only), (combine only) — each repeated R times in
the graph over the rotating input sets — and prints µs per repetition.
"""
import os
import sys
from ctypes import c_void_p
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2512_22036_b200 import EPBuffer, _lib  # noqa: E402
from paper_2512_22036_b200._lib import FS_PHASE_ALL, FS_SRC_ACT  # noqa: E402


def run(cfg: str, R: int = 20, iters: int = 20) -> None:
    hidden, dtype, E, K, T_l, zipf, desc = bench.CONFIGS[cfg]
    dev = torch.device("cuda", 0)
    a, pl = bench.routing_for(cfg, 1, 0)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    buf = EPBuffer(num_experts=E, topk=K, hidden=hidden, dtype=dtype, max_tokens=T_l, with_act_out=False)
    NSET = 2
    xs = [torch.randn(T_l, hidden, device=dev).to(tdt) for _ in range(NSET)]
    outs = [torch.empty(T_l, hidden, device=dev, dtype=tdt) for _ in range(NSET)]
    idx = torch.as_tensor(a.experts, device=dev).contiguous()
    w = torch.as_tensor(a.weights, dtype=torch.float32, device=dev).contiguous()
    plan = buf.r.new_plan(idx, with_masks=False)
    lib = _lib.load()
    h = buf.r.handle
    P_ = lambda t: c_void_p(t.data_ptr())  # noqa: E731
    side = torch.cuda.Stream()
    st = c_void_p(side.cuda_stream)
    lay = (h, P_(idx), idx.element_size(), T_l, P_(plan.row_of), P_(plan.expert_counts),
           P_(plan.expert_offsets), None, None, P_(plan.stats), FS_PHASE_ALL, st)
    disp = [(h, P_(xs[j]), P_(idx), idx.element_size(), P_(plan.row_of), T_l, FS_PHASE_ALL, st) for j in range(NSET)]
    comb = [(h, P_(idx), idx.element_size(), P_(plan.row_of), P_(w), 4, T_l, P_(outs[j]), buf.dtype_code,
             FS_SRC_ACT, 0, FS_PHASE_ALL, st) for j in range(NSET)]

    def body(parts):
        def f():
            for j in range(R):
                if "l" in parts:
                    lib.fs_layout(*lay)
                if "d" in parts:
                    lib.fs_dispatch(*disp[j % NSET])
                if "c" in parts:
                    lib.fs_combine(*comb[j % NSET])
        return f

    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        body("ldc")()
        torch.cuda.synchronize()
        res = {}
        for parts in ("ldc", "dc", "l", "d", "c", "ld"):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                body(parts)()
            for _ in range(3):
                g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(side)
            for _ in range(iters):
                g.replay()
            e1.record(side)
            torch.cuda.synchronize()
            res[parts] = e0.elapsed_time(e1) * 1e3 / (iters * R)
    buf.check()
    print(f"{cfg:12s} " + "  ".join(f"{k}={v:6.2f}" for k, v in res.items())
          + f"   layout marginal={res['ldc'] - res['dc']:.2f} us", flush=True)
    buf.close()


if __name__ == "__main__":
    for c in sys.argv[1:] or ["mixtral", "qwen3", "dsv3", "dsv3_decode"]:
        run(c)
