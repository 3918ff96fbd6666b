"""Benchmark matrix on the GPU (reference bench.py:48-289, §8f next row #2).

Same cells (pattern x seq_len, seq_len = total tokens as the reference's
``generate(pattern, seq_len, ...)``, bench.py:128-132) and variants (fused, baseline =
disaggregated pack/exchange/unpack, planner_off = no dedup, balancer_off =
static groups and the device balancing off — static work striding, no
rotation, ``fs_set_balance``) and the same row fields as the reference
(``ROW_FIELDS``, bench.py:48-63), but the times are CUDA-event measurements
of the kernels on one B200 with the P ranks emulated (``run_exchange``), plus
``latency_us``, ``routed_gbps`` (2·T·K·tb per round trip / time), ``hbm_gbps``
(algorithmic HBM bytes of the emulated round trip, 2·T·tb + 2·T·K·tb, / time)
and ``roofline_frac`` (hbm_gbps / the measured HBM peak).  Rows are emitted as JSON (schema id
``fusco-b200/bench-result/1``, sha256 config fingerprint), CSV or Markdown.

    python -m paper_2512_22036_b200.matrix --topology box8 --seq-lens 4096 8192 \
        --variants fused baseline planner_off --format md
    python -m paper_2512_22036_b200.matrix --topology topo.json --trace captured.json
"""

from __future__ import annotations

import argparse
import csv
import hashlib
import io
import json
import sys
from dataclasses import dataclass, field, replace
from pathlib import Path

import numpy as np

from .routing import GENERATORS, RoutingAssignment, generate, load_trace
from .topology import ClusterTopology, ExpertPlacement, load_topology, preset

SCHEMA_ID = "fusco-b200/bench-result/1"
ROW_FIELDS = (
    "pattern", "seq_len", "variant", "mode", "balancer", "preprocess_s", "rearrange_s", "communicate_s",
    "total_s", "inter_node_bytes", "intra_node_bytes", "intra_gpu_bytes", "rearrange_bytes", "dedup_ratio",
    "latency_us", "routed_gbps", "hbm_gbps", "roofline_frac",
)
DEFAULT_SEQ_LENS = (4096, 8192, 16384, 32768)
VARIANT_ABLATE = {"fused": (), "baseline": ("dcomm", "planner"), "dcomm_off": ("dcomm",),
                  "planner_off": ("planner",), "balancer_off": ("balancer",)}


@dataclass
class BenchConfig:
    topo: ClusterTopology
    placement: ExpertPlacement
    patterns: tuple[str, ...] = tuple(sorted(GENERATORS))
    seq_lens: tuple[int, ...] = DEFAULT_SEQ_LENS
    topk: int = 8
    token_bytes: int = 14336
    dtype: str = "bf16"
    balancer: str = "greedy"
    variants: tuple[str, ...] = ("fused", "baseline", "planner_off", "balancer_off")
    seed: int = 0
    repeats: int = 3
    extra: dict = field(default_factory=dict)
    # a recorded routing (reference bench.py:79-80, 123-130): replaces the
    # generated patterns with one cell of the trace's tokens
    trace: RoutingAssignment | None = None
    trace_label: str = "trace"

    def fingerprint_doc(self) -> dict:
        return {
            "num_nodes": self.topo.num_nodes, "gpus_per_node": self.topo.gpus_per_node,
            "num_experts": self.placement.num_experts, "placement": self.placement.owner.tolist(),
            "patterns": list(self.patterns), "seq_lens": list(self.seq_lens), "topk": self.topk,
            "token_bytes": self.token_bytes, "dtype": self.dtype, "balancer": self.balancer,
            "variants": list(self.variants), "seed": self.seed, "repeats": self.repeats,
            "trace": self.trace_label if self.trace is not None else None,
        }

    def fingerprint(self) -> str:
        return hashlib.sha256(json.dumps(self.fingerprint_doc(), sort_keys=True).encode()).hexdigest()


def cells(cfg: BenchConfig) -> list[tuple[str, int]]:
    if cfg.trace is not None:
        return [(cfg.trace_label, cfg.trace.num_tokens)]
    return [(p, s) for p in cfg.patterns for s in cfg.seq_lens]


def cell_assignment(cfg: BenchConfig, index: int, pattern: str, seq_len: int):
    """Per-cell routing: seq_len tokens in total, SeedSequence((seed, index))
    as the reference (bench.py:128-132); the recorded trace when one is given."""
    if cfg.trace is not None:
        return cfg.trace
    rng = np.random.default_rng(np.random.SeedSequence((cfg.seed, index)))
    return generate(pattern, seq_len, cfg.topk, cfg.topo, cfg.placement, rng)


def hbm_peak_gbs() -> float:
    p = Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"])
    return 6650.0  # B200_PROFILING.md fallback


def graph_time_exchange(a, topo, placement, token_bytes, ablate=(), dtype="bf16", iters=10, device=None):
    """Device time of the fused round trip of every emulated rank, replayed
    as three CUDA graphs (layout / dispatch / combine over all ranks and
    phases) so the host launch cost of P x 2 phases x 3 calls is not counted.
    Returns mean seconds (layout, dispatch, combine)."""
    import torch

    from .api import _open_session, make_token_payloads
    from .engine import FS_ACC_F32, FS_SRC_ACT, dtype_code

    tdt, code = dtype_code(dtype)
    sess = _open_session(a, topo, placement, token_bytes, ablate, with_act_out=False, device=device)
    try:
        cl, dev = sess.cluster, sess.dev
        payloads = make_token_payloads(a.num_tokens, token_bytes, 0)
        xs = [torch.as_tensor(payloads[i], device=dev).contiguous() for i in sess.ids]
        ws = [torch.as_tensor(a.weights[i], dtype=torch.float32, device=dev).contiguous() for i in sess.ids]
        outs = [torch.empty((i.size, token_bytes), dtype=torch.uint8, device=dev).view(tdt) for i in sess.ids]
        plans = cl.layout(sess.idx, with_masks=False)
        stages = (lambda: cl.layout_into(plans),
                  lambda: cl.dispatch(xs, plans),
                  lambda: cl.combine(plans, ws, outs, dtype_code=code, src=FS_SRC_ACT, acc=FS_ACC_F32))
        for f in stages[1:]:
            f()
        cl.check()
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        graphs = []
        with torch.cuda.stream(side):
            for f in stages:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=side):
                    f()
                graphs.append(g)
        torch.cuda.current_stream(dev).wait_stream(side)
        for _ in range(2):
            for g in graphs:
                g.replay()
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(iters)]
        torch.cuda.synchronize(dev)
        for e in ev:
            e[0].record()
            for i, g in enumerate(graphs):
                g.replay()
                e[i + 1].record()
        torch.cuda.synchronize(dev)
        cl.check()
        return tuple(sum(e[i].elapsed_time(e[i + 1]) for e in ev) / iters * 1e-3 for i in range(3))
    finally:
        sess.close()


def run_cell(cfg: BenchConfig, index: int, pattern: str, seq_len: int) -> list[dict]:
    from .api import dedup_ratio, run_exchange

    a = cell_assignment(cfg, index, pattern, seq_len)
    ratio = dedup_ratio(a, cfg.topo, cfg.placement)
    peak = hbm_peak_gbs()
    rows = []
    for variant in cfg.variants:
        ablate = VARIANT_ABLATE[variant]
        fused = "dcomm" not in ablate
        best = None
        for _ in range(1 if fused else max(1, cfg.repeats)):
            r = run_exchange(a, cfg.topo, cfg.placement, cfg.token_bytes, payload_seed=cfg.seed, ablate=ablate,
                             balancer=cfg.balancer, materialize=False, dtype=cfg.dtype, acc="f32")
            if best is None or r.total_s < best.total_s:
                best = r
        d, c = best.dispatch_report, best.combine_report
        if fused:  # kernel time without the emulation's host launch cost (the eager pack/a2a/unpack
            #        baseline keeps its eager times: its host syncs are part of that design)
            t_lay, t_disp, t_comb = graph_time_exchange(a, cfg.topo, cfg.placement, cfg.token_bytes, ablate,
                                                        cfg.dtype, iters=max(3, 5 * cfg.repeats))
            d = replace(d, preprocess_s=t_lay, rearrange_s=0.0, communicate_s=t_disp)
            c = replace(c, preprocess_s=0.0, rearrange_s=0.0, communicate_s=t_comb)
        total = d.total_s + c.total_s
        routed = 2.0 * a.num_tokens * a.topk * cfg.token_bytes
        hbm = routed + 2.0 * a.num_tokens * cfg.token_bytes
        gbs = hbm / total / 1e9 if total > 0 else 0.0
        rows.append({
            "pattern": pattern, "seq_len": seq_len, "variant": variant, "mode": "gpu-graph" if fused else "gpu-eager",
            "balancer": "static" if "balancer" in ablate else cfg.balancer,
            "preprocess_s": d.preprocess_s + c.preprocess_s, "rearrange_s": d.rearrange_s + c.rearrange_s,
            "communicate_s": d.communicate_s + c.communicate_s, "total_s": total,
            "inter_node_bytes": int(d.inter_node_bytes + c.inter_node_bytes),
            "intra_node_bytes": int(d.intra_node_bytes + c.intra_node_bytes),
            "intra_gpu_bytes": int(d.intra_gpu_bytes + c.intra_gpu_bytes),
            "rearrange_bytes": int(d.rearrange_bytes + c.rearrange_bytes), "dedup_ratio": float(ratio),
            "latency_us": total * 1e6, "routed_gbps": routed / total / 1e9 if total > 0 else 0.0,
            "hbm_gbps": gbs, "roofline_frac": gbs / peak,
        })
    return rows


def run_matrix(cfg: BenchConfig) -> dict:
    rows = []
    for i, (p, s) in enumerate(cells(cfg)):
        rows.extend(run_cell(cfg, i, p, s))
    return {"schema": SCHEMA_ID, "fingerprint": cfg.fingerprint(),
            "config": {**cfg.fingerprint_doc(), "device": "B200, ranks emulated on one GPU", **cfg.extra},
            "rows": rows}


def validate_result(doc: dict) -> None:
    """Structural check of a result document (the reference ships a JSON
    schema, schemas/bench_result.schema.json; same required fields)."""
    if doc.get("schema") != SCHEMA_ID or len(doc.get("fingerprint", "")) != 64:
        raise ValueError("not a fusco-b200 bench result")
    for row in doc["rows"]:
        missing = set(ROW_FIELDS) - set(row)
        if missing:
            raise ValueError(f"row missing {sorted(missing)}")
        if row["variant"] not in VARIANT_ABLATE:
            raise ValueError(f"unknown variant {row['variant']}")
        if row["dedup_ratio"] < 1 or min(row[k] for k in ROW_FIELDS[5:14]) < 0:
            raise ValueError("negative time/byte counter or dedup ratio < 1")


def render(doc: dict, fmt: str) -> str:
    rows = doc["rows"]
    if fmt == "json":
        return json.dumps(doc, indent=1, sort_keys=True) + "\n"
    if fmt == "csv":
        buf = io.StringIO()
        w = csv.DictWriter(buf, fieldnames=list(ROW_FIELDS), lineterminator="\n")
        w.writeheader()
        for r in rows:
            w.writerow({k: r[k] for k in ROW_FIELDS})
        return buf.getvalue()
    if fmt == "md":
        cols = ("pattern", "seq_len", "variant", "latency_us", "routed_gbps", "roofline_frac", "rearrange_s",
                "communicate_s", "inter_node_bytes", "rearrange_bytes", "dedup_ratio")
        out = [f"<!-- {doc['schema']} fingerprint {doc['fingerprint']} -->",
               "| " + " | ".join(cols) + " |", "|" + "---|" * len(cols)]
        for r in rows:
            out.append("| " + " | ".join(f"{r[c]:.4g}" if isinstance(r[c], float) else str(r[c]) for c in cols) + " |")
        return "\n".join(out) + "\n"
    raise ValueError(f"unknown format {fmt!r}")


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--topology", "--preset", dest="topology", default="box8",
                    help="topology preset (box8, test, large) or path to a topology JSON file (bench.py:291-298)")
    ap.add_argument("--trace", default=None,
                    help="routing trace JSON (save_trace format); replaces the generated patterns (bench.py:343-346)")
    ap.add_argument("--patterns", nargs="+", default=sorted(GENERATORS))
    ap.add_argument("--seq-lens", nargs="+", type=int, default=list(DEFAULT_SEQ_LENS), help="total tokens")
    ap.add_argument("--topk", type=int, default=8)
    ap.add_argument("--token-bytes", type=int, default=14336)
    ap.add_argument("--variants", nargs="+", default=["fused", "baseline", "planner_off", "balancer_off"],
                    choices=sorted(VARIANT_ABLATE))
    ap.add_argument("--balancer", default="greedy", choices=["greedy", "static", "optimal"])
    ap.add_argument("--format", default="md", choices=["json", "csv", "md"])
    ap.add_argument("--out", default="-")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--dump-plan", default=None, metavar="PATH",
                    help="also write the first cell's device plans as plan_to_json documents (bench.py:399-421)")
    args = ap.parse_args(argv)
    try:
        if Path(args.topology).exists():
            topo, pl = load_topology(args.topology)
        else:
            topo, pl = preset(args.topology)
    except (OSError, ValueError, KeyError) as exc:
        print(f"error: topology {args.topology!r}: {exc}", file=sys.stderr)
        return 2
    trace, label, token_bytes, topk = None, "trace", args.token_bytes, args.topk
    if args.trace:
        try:
            trace, token_bytes = load_trace(args.trace)
        except (OSError, ValueError, KeyError) as exc:
            print(f"error: trace {args.trace!r}: {exc}", file=sys.stderr)
            return 2
        label, topk = Path(args.trace).name, trace.topk
    cfg = BenchConfig(topo, pl, tuple(args.patterns), tuple(args.seq_lens), topk, token_bytes,
                      balancer=args.balancer, variants=tuple(args.variants), seed=args.seed, repeats=args.repeats,
                      trace=trace, trace_label=label)
    if args.dump_plan:
        from .api import run_exchange
        from .wire import plan_to_json

        first = cells(cfg)[0]
        res = run_exchange(cell_assignment(cfg, 0, *first), cfg.topo, cfg.placement, cfg.token_bytes,
                           balancer=cfg.balancer, materialize=False, dtype=cfg.dtype, acc="f32")
        m = cfg.topo.gpus_per_node
        with open(args.dump_plan, "w") as fh:
            json.dump({"dispatch": plan_to_json(res.dispatch_plan, m), "combine": plan_to_json(res.combine_plan, m)},
                      fh, indent=2, sort_keys=True)
            fh.write("\n")
    doc = run_matrix(cfg)
    validate_result(doc)
    text = render(doc, args.format)
    if args.out == "-":
        sys.stdout.write(text)
    else:
        with open(args.out, "w") as fh:
            fh.write(text)
    return 0


if __name__ == "__main__":
    sys.exit(main())
