"""Per-kernel NVLink bytes of the shuffle on P real GPUs, counted by ncu.

ncu cannot wrap a multi-rank run (kernels of different ranks wait on each
other).  Here ONE process drives P GPUs (rank r on cuda:r, peer access
enabled, ``EmulatedCluster(devices=...)``) and launches the phases the way
the single-GPU emulation does — LOCAL of every rank, then REMOTE — so no
kernel waits on one that has not run, and every kernel moves its real bytes
over NVLink.  ncu then counts each kernel's NVLink traffic on its own GPU:
the dispatch push (LOCAL) as the pusher's TX, the combine pull (REMOTE) as
the puller's RX.

    python tools/ncu_nvlink.py --config dsv3 --gpus 2            # plain run (must exit 0 first)
    ncu --metrics gpu__time_duration.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,\\
dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file L.csv \\
        python tools/ncu_nvlink.py --config dsv3 --gpus 2
    python tools/ncu_nvlink.py --config dsv3 --gpus 2 --summarize L.csv   # -> JSON table
"""

from __future__ import annotations

import argparse
import csv
import json
import sys
from collections import defaultdict
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402

FS_NAME = {"layout_kernel": "fs_layout", "dispatch_kernel": "fs_dispatch", "dispatch_tma_kernel": "fs_dispatch",
           "combine_kernel": "fs_combine", "combine_tma_kernel": "fs_combine", "combine_k2_kernel": "fs_combine"}


def run(cfg: str, P: int, iters: int, seed: int) -> None:
    import torch

    from paper_2512_22036_b200.engine import EmulatedCluster

    hidden, dtype, E, K, T_l, zipf, desc = bench.CONFIGS[cfg]
    a, pl = bench.routing_for(cfg, P, seed)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    tb = hidden * (2 if dtype == "bf16" else 4)
    ids = [np.flatnonzero(a.source == s) for s in range(P)]
    devs = [torch.device("cuda", r) for r in range(P)]
    with EmulatedCluster(P, E, K, tb, T_l, owner=pl.owner, devices=devs) as cl:
        xs = [torch.randn(i.size, hidden, device=d).to(tdt) for i, d in zip(ids, devs)]
        idx = [torch.as_tensor(a.experts[i], device=d) for i, d in zip(ids, devs)]
        ws = [torch.as_tensor(a.weights[i], dtype=torch.float32, device=d) for i, d in zip(ids, devs)]
        outs = [torch.empty_like(x) for x in xs]
        for _ in range(iters):
            plans = cl.layout(idx, with_masks=False)
            cl.dispatch(xs, plans, ws=ws)  # router weights at dispatch: owner pre-reduction where enabled
            cl.combine(plans, ws, outs, dtype_code=1 if dtype == "bf16" else 0)
        cl.check()
        for s in range(P):  # identity experts: the round trip returns x (weights sum to 1)
            ref = (xs[s].float() * ws[s].sum(1, keepdim=True)).to(tdt).float()
            if not torch.allclose(outs[s].float(), ref, rtol=2.0**-7, atol=2e-2):
                raise SystemExit(f"round trip failed on rank {s}")
    print(f"ncu_nvlink: {cfg} P={P} iters={iters} ok", flush=True)


def summarize(cfg: str, P: int, path: str, seed: int) -> dict:
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if "Kernel Name" in r)
    hi = rows.index(hdr)
    col = {k: hdr.index(k) for k in ("ID", "Device", "Kernel Name", "Metric Name", "Metric Value")}
    launches: dict[int, dict] = {}
    for r in rows[hi + 1:]:
        if len(r) != len(hdr):
            continue
        name = r[col["Kernel Name"]].split("(")[0].replace("void ", "").replace("fusco::", "").split("<")[0].strip()
        if name not in FS_NAME:
            continue
        lid = int(r[col["ID"]])
        d = launches.setdefault(lid, {"kernel": FS_NAME[name], "device": int(r[col["Device"]]), "m": {}})
        d["m"][r[col["Metric Name"]]] = float(r[col["Metric Value"]].replace(",", ""))
    # phase of each launch: per (device, kernel) the launches alternate LOCAL, REMOTE
    seq = defaultdict(int)
    agg = defaultdict(lambda: defaultdict(list))
    for lid in sorted(launches):
        d = launches[lid]
        key = (d["device"], d["kernel"])
        phase = "local" if seq[key] % 2 == 0 else "remote"
        seq[key] += 1
        for m, v in d["m"].items():
            agg[(d["kernel"], phase, d["device"])][m].append(v)
    hidden, dtype, E, K, T_l, zipf, desc = bench.CONFIGS[cfg]
    tb = hidden * (2 if dtype == "bf16" else 4)
    a, pl = bench.routing_for(cfg, P, seed)
    tr = bench.traffic(a.experts, a.source, pl.owner, P, tb, T_l)
    out = {"config": cfg, "workload": desc, "P": P, "source": "ncu nvltx__bytes_data_user / nvlrx__bytes_data_user "
           "per launch (32 B granularity), phased single-process run on P GPUs", "kernels": []}
    for (kern, phase, dev), ms in sorted(agg.items()):
        mean = {m: float(np.mean(v)) for m, v in ms.items()}
        row = {"kernel": kern, "phase": phase, "gpu": dev, "launches": len(next(iter(ms.values()))),
               "us": mean.get("gpu__time_duration.sum", 0.0) / 1e3,
               "nvl_tx_bytes": mean.get("nvltx__bytes_data_user.sum"), "nvl_rx_bytes": mean.get("nvlrx__bytes_data_user.sum"),
               "dram_bytes": mean.get("dram__bytes_read.sum", 0.0) + mean.get("dram__bytes_write.sum", 0.0)}
        if kern == "fs_dispatch" and phase == "local":
            row["alg_tx_bytes"] = float(tr["d_eg"][dev])   # deduplicated push to the other ranks
        if kern == "fs_combine" and phase == "remote":
            row["alg_rx_bytes"] = float(tr["c_in"][dev])   # rows pulled from the other ranks
            row["alg_rx_bytes_owner_reduce"] = float(tr["c_in_red"][dev])  # with owner pre-reduction
        if row["us"] > 0 and row["nvl_tx_bytes"] is not None:
            row["nvl_tx_gbps"] = row["nvl_tx_bytes"] / (row["us"] * 1e-6) / 1e9
            row["nvl_rx_gbps"] = row["nvl_rx_bytes"] / (row["us"] * 1e-6) / 1e9
        out["kernels"].append(row)
    return out


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="dsv3", choices=sorted(bench.CONFIGS))
    ap.add_argument("--gpus", type=int, default=2)
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--summarize", default=None, metavar="CSV")
    args = ap.parse_args()
    if args.summarize:
        print(json.dumps(summarize(args.config, args.gpus, args.summarize, args.seed), indent=1))
        return 0
    run(args.config, args.gpus, args.iters, args.seed)
    return 0


if __name__ == "__main__":
    sys.exit(main())
