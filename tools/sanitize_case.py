"""Small emulated shuffle for compute-sanitizer (4 ranks on one GPU, both engines)."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import shuffle_oracle as O  # noqa: E402
from paper_2512_22036_b200 import box, gen_realworld, round_robin_placement  # noqa: E402
from paper_2512_22036_b200.engine import EmulatedCluster  # noqa: E402

torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
P, E, K, H, T_l = 4, 32, 4, 512, 96
for eng in ("warp", "tma"):
    os.environ["FUSCO_DISPATCH"] = eng
    os.environ["FUSCO_COMBINE"] = eng
    topo = box(P)
    pl = round_robin_placement(E, topo)
    a = gen_realworld(P * T_l, K, topo, pl, seed=1, zipf_s=0.9)
    payload = O.encode(np.random.default_rng(0).standard_normal((a.num_tokens, H)).astype(np.float32), "bf16")
    ids = [np.flatnonzero(a.source == s) for s in range(P)]
    with EmulatedCluster(P, E, K, H * 2, T_l, owner=pl.owner, device=dev) as cl:
        for it in range(2):
            plans = cl.layout([torch.as_tensor(a.experts[i], device=dev) for i in ids])
            cl.dispatch([torch.as_tensor(payload[i], device=dev).contiguous() for i in ids], plans)
            outs = [torch.empty((i.size, H), dtype=torch.bfloat16, device=dev) for i in ids]
            cl.combine(plans, [torch.as_tensor(a.weights[i], dtype=torch.float32, device=dev) for i in ids], outs,
                       dtype_code=1)
            cl.check()
    # single rank (cluster planner + pipelined combine paths)
    os.environ["FUSCO_LAYOUT"] = "cluster"
    with EmulatedCluster(1, 8, 2, H * 2, 300, device=dev) as cl:
        idx = torch.as_tensor(gen_realworld(300, 2, box(1), round_robin_placement(8, box(1)), seed=2).experts,
                              device=dev)
        plans = cl.layout([idx])
        x = torch.randn(300, H, device=dev).to(torch.bfloat16)
        cl.dispatch([x], plans)
        out = torch.empty_like(x)
        cl.combine(plans, [torch.full((300, 2), 0.5, device=dev)], [out], dtype_code=1)
        cl.check()
    os.environ.pop("FUSCO_LAYOUT")
torch.cuda.synchronize()
print("sanitize case OK")
