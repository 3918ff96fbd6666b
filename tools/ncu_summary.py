"""Summarise ncu captures into profiles/ (committed evidence).

    python tools/ncu_summary.py <tag> <config> <n_gpus> <launches.csv> <prof.ncu-rep> [more reps...]

Writes profiles/<tag>_<config>_n<N>.md (launch list + key full-set metrics
per kernel) and merges per-launch DRAM traffic into profiles/ncu_traffic.json
(key "<config>/n<N>/<fs_kernel>", read by bench.py for roofline.traffic).
"""
import csv
import json
import statistics
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
PROF = ROOT / "profiles"
FS_NAME = {"layout_kernel": "fs_layout", "dispatch_kernel": "fs_dispatch", "dispatch_tma_kernel": "fs_dispatch",
           "combine_kernel": "fs_combine", "combine_tma_kernel": "fs_combine",
           "combine_k2_kernel": "fs_combine"}
METRICS = [
    ("gpu__time_duration.sum", "duration", "us", 1e-3),
    ("dram__bytes_read.sum", "DRAM read", "MB", 1e-6),
    ("dram__bytes_write.sum", "DRAM write", "MB", 1e-6),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput", "% of peak", 1),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput", "%", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy", "%", 1),
    ("launch__registers_per_thread", "registers/thread", "", 1),
    ("launch__grid_size", "grid", "CTAs", 1),
    ("launch__block_size", "block", "threads", 1),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/CTA", "B", 1),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe", "%", 1),
]


def short(name: str) -> str:
    n = name.split("(")[0].replace("void ", "").replace("fusco::", "").strip()
    return n.split("<")[0]


def launch_list(path):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if "Kernel Name" in r)
    hi = rows.index(hdr)
    K, M, V = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: defaultdict(list))
    for r in rows[hi + 1:]:
        if len(r) == len(hdr):
            agg[short(r[K])][r[M]].append(float(r[V].replace(",", "")))
    return agg


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    scale = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "second": 1e9,  # -> ns
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "Kbyte/block": 1e3}  # -> bytes
    res = defaultdict(list)
    for d in data:
        rec = {}
        for h, u, v in zip(hdr, units, d):
            if u in scale:
                try:
                    v = str(float(v.replace(",", "")) * scale[u])
                except ValueError:
                    pass
            rec[h] = v
        res[short(rec["Kernel Name"])].append(rec)
    return res


def main():
    tag, cfg, n = sys.argv[1], sys.argv[2], int(sys.argv[3])
    launches, reps = sys.argv[4], sys.argv[5:]
    PROF.mkdir(exist_ok=True)
    lines = [f"# ncu summary: {tag}, config `{cfg}`, {n} GPU(s)", "",
             "Launch list (`--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
             "--clock-control none`; cold-cache, serialised — compare shares, not absolutes):", "",
             "| kernel | launches | median us | share | DRAM read MB | DRAM write MB |", "|---|---|---|---|---|---|"]
    agg = launch_list(launches)
    tot = sum(statistics.median(m["gpu__time_duration.sum"]) for m in agg.values())
    traffic_file = PROF / "ncu_traffic.json"
    traffic = json.loads(traffic_file.read_text()) if traffic_file.exists() else {}
    for k, m in agg.items():
        t = statistics.median(m["gpu__time_duration.sum"])
        rd = statistics.median(m.get("dram__bytes_read.sum", [0]))
        wr = statistics.median(m.get("dram__bytes_write.sum", [0]))
        lines.append(f"| {k} | {len(m['gpu__time_duration.sum'])} | {t / 1e3:.2f} | {100 * t / tot:.1f}% | "
                     f"{rd / 1e6:.2f} | {wr / 1e6:.2f} |")
        if k in FS_NAME:
            traffic[f"{cfg}/n{n}/{FS_NAME[k]}"] = rd + wr
    traffic_file.write_text(json.dumps(traffic, indent=1, sort_keys=True) + "\n")
    for rep in reps:
        lines += ["", f"Full set (`--set full`), `{Path(rep).name}`:", ""]
        raw = raw_metrics(rep)
        kernels = sorted(raw)
        lines.append("| metric | " + " | ".join(kernels) + " |")
        lines.append("|---|" + "---|" * len(kernels))
        for key, label, unit, scale in METRICS:
            vals = []
            for k in kernels:
                v = raw[k][0].get(key)
                try:
                    vals.append(f"{float(v.replace(',', '')) * scale:.2f}")
                except (AttributeError, ValueError):
                    vals.append("-")
            lines.append(f"| {label} ({unit}) | " + " | ".join(vals) + " |")
    out = PROF / f"{tag}_{cfg}_n{n}.md"
    out.write_text("\n".join(lines) + "\n")
    print(out)


if __name__ == "__main__":
    main()
