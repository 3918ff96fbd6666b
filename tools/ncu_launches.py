"""Summarise an ncu launch-list CSV (gpu__time_duration + dram bytes per kernel)."""
import csv
import statistics
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Kernel Name" in r)
hi = rows.index(hdr)
K, M, V = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = defaultdict(lambda: defaultdict(list))
for r in rows[hi + 1:]:
    if len(r) != len(hdr):
        continue
    name = r[K].split("(")[0].replace("void ", "").replace("fusco::", "")
    agg[name][r[M]].append(float(r[V].replace(",", "")))
for name, m in agg.items():
    t = m.get("gpu__time_duration.sum", [0])
    rd = m.get("dram__bytes_read.sum", [0])
    wr = m.get("dram__bytes_write.sum", [0])
    print(f"{name[:40]:40s} n={len(t):3d} median {statistics.median(t) / 1e3:8.2f} us  "
          f"dram rd {statistics.median(rd) / 1e6:8.2f} MB wr {statistics.median(wr) / 1e6:8.2f} MB")
