"""Markdown table of multi-GPU bench lines: python tools/multi_table.py gpurun_out/bench_n*_auto_auto.log"""
import json
import sys

print("| N | config | step us | layout us | dispatch us | combine us | floor dispatch us | floor combine us "
      "| step/floor | NVLink GB/s/GPU dispatch | combine |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
rows = []
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        continue
    k, t = d["kernel_us"], d["t_min_us"]
    nv = d.get("nvlink_gbps_per_gpu") or {}
    rows.append((d["n_gpus"], d["config"].get("workload", "")[:40], d))
for n, _, d in sorted(rows, key=lambda r: (r[0], r[1])):
    k, t = d["kernel_us"], d["t_min_us"]
    nv = d.get("nvlink_gbps_per_gpu") or {}
    name = d["config"].get("name") or d["config"]["workload"].split(":")[0]
    print(f"| {n} | {name} | {d['latency_us']:.1f} | {k['fs_layout']:.1f} | {k['fs_dispatch']:.1f} | "
          f"{k['fs_combine']:.1f} | {t['fs_dispatch']:.1f} | {t['fs_combine']:.1f} | "
          f"{(t['fs_dispatch'] + t['fs_combine']) / d['latency_us']:.2f} | {nv.get('dispatch', 0):.0f} | "
          f"{nv.get('combine', 0):.0f} |")
