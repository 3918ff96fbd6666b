"""Print the hottest SASS instructions (warp-stall samples) of one kernel
from `ncu -i rep --page source --csv -k <kernel>` output."""
import csv
import subprocess
import sys

rep, kernel = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", kernel],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
# several launches may be listed: keep the first one only
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
end = starts[1] if len(starts) > 1 else len(rows)
hdr = rows[starts[0] + 1]
ci = hdr.index("Warp Stall Sampling (All Samples)")
si = hdr.index("Source")
data = [r for r in rows[starts[0] + 2 : end] if len(r) == len(hdr)]
tot = sum(float(r[ci] or 0) for r in data) or 1
print(f"{kernel}: {len(data)} SASS lines, {tot:.0f} samples")
order = sorted(range(len(data)), key=lambda i: -float(data[i][ci] or 0))[:n]
for i in sorted(order):
    r = data[i]
    print(f"{i:5d} {float(r[ci]):7.0f} {100 * float(r[ci]) / tot:5.1f}%  {r[si].strip()[:100]}")
