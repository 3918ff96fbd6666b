"""Phase times of the P > 1 shuffle on P real GPUs, one process (CUDA events).

    python tools/push_probe.py --config mixtral --gpus 2 [--iters 20]

Drives P GPUs from one process (``EmulatedCluster(devices=...)``, rank r on
cuda:r) and times each phase per GPU with CUDA events on the launching
stream: the dispatch LOCAL phase (the push: every rank's push runs at once,
so every link carries both directions) and REMOTE phase (block arrival +
receiver fan-out), the combine REMOTE phase (the pull).  Prints one JSON
line: per-phase medians per GPU and the push / pull NVLink GB/s against the
algorithmic bytes.  Used for A/B of dispatch variants
(env knobs, FUSCO_LIB builds) without the planner and handshakes around them.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def main() -> int:
    import torch

    from paper_2512_22036_b200 import _lib
    from paper_2512_22036_b200.engine import EmulatedCluster

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mixtral", choices=sorted(bench.CONFIGS))
    ap.add_argument("--gpus", type=int, default=2)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--tag", default="")
    ap.add_argument("--push-only", action="store_true",
                    help="time only the push (LOCAL phase); for builds without block accounting")
    args = ap.parse_args()
    P = args.gpus
    hidden, dtype, E, K, T_l, zipf, desc = bench.CONFIGS[args.config]
    a, pl = bench.routing_for(args.config, P, 0)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    tb = hidden * (2 if dtype == "bf16" else 4)
    ids = [np.flatnonzero(a.source == s) for s in range(P)]
    devs = [torch.device("cuda", r) for r in range(P)]
    tr = bench.traffic(a.experts, a.source, pl.owner, P, tb, T_l)
    L, R = _lib.FS_PHASE_LOCAL, _lib.FS_PHASE_REMOTE
    times = {k: [[] for _ in range(P)] for k in ("push", "fanout", "c_local", "pull")}
    with EmulatedCluster(P, E, K, tb, T_l, owner=pl.owner, devices=devs) as cl:
        xs = [torch.randn(i.size, hidden, device=d).to(tdt) for i, d in zip(ids, devs)]
        idx = [torch.as_tensor(a.experts[i], device=d) for i, d in zip(ids, devs)]
        ws = [torch.as_tensor(a.weights[i], dtype=torch.float32, device=d) for i, d in zip(ids, devs)]
        outs = [torch.empty_like(x) for x in xs]

        def phase(name, fn):
            ev = []
            for r in range(P):
                with torch.cuda.device(devs[r]):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    fn(r)
                    e1.record()
                    ev.append((e0, e1))
            for r in range(P):
                torch.cuda.synchronize(devs[r])
            if name:
                for r, (e0, e1) in enumerate(ev):
                    times[name][r].append(e0.elapsed_time(e1) * 1e3)

        for it in range(args.iters + 3):
            plans = cl.layout(idx, with_masks=False)
            keep = it >= 3
            phase("push" if keep else None, lambda r: cl.ranks[r].dispatch(xs[r], plans[r], L))
            if args.push_only:
                continue
            phase("fanout" if keep else None, lambda r: cl.ranks[r].dispatch(xs[r], plans[r], R))
            phase("c_local" if keep else None,
                  lambda r: cl.ranks[r].combine(plans[r], ws[r], outs[r], dtype_code=1, phase=L))
            phase("pull" if keep else None,
                  lambda r: cl.ranks[r].combine(plans[r], ws[r], outs[r], dtype_code=1, phase=R))
        if not args.push_only:
            cl.check()
    med = {k: [float(np.median(v)) if v else 0.0 for v in vs] for k, vs in times.items()}
    out = {"config": args.config, "P": P, "tag": args.tag, "us": {k: [round(x, 1) for x in v] for k, v in med.items()},
           "push_gbps": [round(float(tr["d_eg"][r]) / (med["push"][r] * 1e-6) / 1e9, 1) for r in range(P)],
           "pull_gbps": [round(float(tr["c_in"][r]) / (med["pull"][r] * 1e-6) / 1e9, 1) if med["pull"][r] else None
                         for r in range(P)],
           "push_mb": [round(float(tr["d_eg"][r]) / 1e6, 2) for r in range(P)],
           "pull_mb": [round(float(tr["c_in"][r]) / 1e6, 2) for r in range(P)]}
    print(json.dumps(out), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
