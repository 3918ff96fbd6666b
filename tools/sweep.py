"""Run bench.py variants (env knobs x args) and print one compact line each.

    python tools/sweep.py <config>[,<config>...] "<label>|ENV=V,ENV=V|--arg v" ...
"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
out_dir = ROOT / "gpurun_out"
out_dir.mkdir(exist_ok=True)
configs = sys.argv[1].split(",")
for cfg in configs:
    for spec in sys.argv[2:]:
        label, envs, args = (spec.split("|") + ["", ""])[:3]
        env = dict(os.environ)
        for kv in filter(None, envs.split(",")):
            k, v = kv.split("=", 1)
            env[k] = v
        cmd = [sys.executable, str(ROOT / "bench.py"), "--config", cfg, "--steps", "100", "--warmup", "10",
               "--no-cpu-baseline", "--no-e2e", "--graph", *args.split()]
        log = out_dir / f"sweep_{cfg}_{label}.log"
        try:
            res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=300)
            log.write_text(res.stdout + res.stderr)
            d = json.loads(res.stdout.strip().splitlines()[-1])
            k = {n: round(v, 1) for n, v in d["kernel_us"].items()}
            print(f"{cfg:12s} {label:14s} {d['latency_us']:8.1f} us  {k}  tmin {d['t_min_us']}  "
                  f"frac {d['roofline']['frac']:.3f}", flush=True)
        except Exception as exc:  # noqa: BLE001
            print(f"{cfg:12s} {label:14s} FAILED {exc}", flush=True)
