"""Tabulate the ncu NVLink counter JSONs (tools/ncu_nvlink.py --summarize) into profiles/r2_nvlink_counters.md.

    python tools/nvl_table.py profiles/r2_nvl_counters_*.json > profiles/r2_nvlink_counters.md
"""
import json
import statistics
import sys

rows = []
for f in sorted(sys.argv[1:]):
    d = json.load(open(f))
    by = {}
    for k in d["kernels"]:
        if k["kernel"] == "fs_layout" or k["us"] < 10:
            continue
        by.setdefault((k["kernel"], k["phase"]), []).append(k)
    for (kern, ph), ks in sorted(by.items()):
        link = [k["nvl_tx_bytes"] if ph == "local" else k["nvl_rx_bytes"] for k in ks]
        alg = [k.get("alg_tx_bytes", k.get("alg_rx_bytes")) for k in ks]
        red = [k.get("alg_rx_bytes_owner_reduce") for k in ks]
        us = [k["us"] for k in ks]
        gbps = [b / t / 1e3 for b, t in zip(link, us)]
        dram = [k["dram_bytes"] for k in ks]
        ratio = "—" if alg[0] is None else f"{sum(link) / sum(alg):.4f}"
        rred = "—" if red[0] is None else f"{statistics.mean(red) / 1e6:.2f} ({sum(link) / sum(red):.4f})"
        rows.append((d["config"], d["P"], kern, ph, statistics.mean(us), statistics.mean(link) / 1e6,
                     None if alg[0] is None else statistics.mean(alg) / 1e6, ratio,
                     statistics.mean(gbps), statistics.mean(dram) / 1e6, rred))
print("| config | P | kernel | phase | µs (mean over GPUs) | NVLink bytes/GPU (MB, counter) | algorithmic (MB) | counter / algorithmic | owner-reduced algorithmic (MB, counter / it) | NVLink GB/s/GPU | DRAM MB/GPU |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for r in rows:
    alg = "—" if r[6] is None else f"{r[6]:.2f}"
    print(f"| {r[0]} | {r[1]} | {r[2]} | {r[3]} ({'push, TX' if r[3] == 'local' and r[2] == 'fs_dispatch' else 'owner pre-reduction, HBM' if r[3] == 'local' else 'pull, RX' if r[2] == 'fs_combine' else 'fan-out, HBM'}) | {r[4]:.1f} | {r[5]:.2f} | {alg} | {r[7]} | {r[10]} | {r[8]:.0f} | {r[9]:.1f} |")
