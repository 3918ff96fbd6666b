"""Calibrate the NVML NVLink byte counters against a known peer copy.

    python tools/nvlink_probe.py [--mib 4096]

Copies N MiB from cuda:0 to cuda:1 (peer copy over NVLink) and prints both
GPUs' counter deltas, data and raw (with protocol overhead).  Expect
TX(0) ~= RX(1) ~= N.  (The engine's own SM movers are counted by bench.py
at N > 1 around its timed region.)
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main() -> int:
    import torch

    from paper_2512_22036_b200.nvlink import NvlinkCounters

    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=4096)
    args = ap.parse_args()
    n = args.mib << 20
    if torch.cuda.device_count() < 2:
        print(json.dumps({"error": "needs 2 GPUs"}))
        return 0
    c = [NvlinkCounters(torch.device("cuda", i)) for i in range(2)]
    out = {"links": [x.links for x in c], "pci": [x.pci for x in c], "mode": [x.mode for x in c],
           "rejected": [x.errors for x in c]}
    a = torch.empty(n, dtype=torch.uint8, device="cuda:0").fill_(1)
    b = torch.empty(n, dtype=torch.uint8, device="cuda:1")
    torch.cuda.synchronize("cuda:0")
    torch.cuda.synchronize("cuda:1")
    for rep in range(2):
        for x in c:
            x.start()
        for _ in range(4):
            b.copy_(a)
        torch.cuda.synchronize("cuda:0")
        torch.cuda.synchronize("cuda:1")
        got = [x.stop() for x in c]
        out[f"ce_copy_x4_{rep}"] = {f"gpu{i}": {"tx": got[i][0], "rx": got[i][1]} for i in range(2)}
    try:
        import subprocess

        out["nvidia_smi_nvlink_gt_d"] = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", "0"],
                                                       capture_output=True, text=True, timeout=30).stdout[-1500:]
    except Exception as e:  # noqa: BLE001
        out["nvidia_smi_nvlink_gt_d"] = repr(e)
    out["bytes_per_copy"] = n
    print(json.dumps(out, indent=1))
    return 0


if __name__ == "__main__":
    sys.exit(main())
