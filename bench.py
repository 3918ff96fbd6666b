"""Benchmark: MoE dispatch+combine (Fusco shuffle) on 1-8 B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--impl fusco|reference]

N > 1 is launched by torchrun (one process per GPU, NCCL bootstrap only).
A step = one pass of the hot path over one batch: on-device layout planner
(fs_layout) + dispatch (fs_dispatch) + combine (fs_combine), identity expert
(combine pulls the dispatched rows straight back), fp32 accumulation, bf16
payloads.  Inputs are resident in HBM for ``value``; ``e2e`` repeats the
step through the public API with pinned host buffers and the H2D/D2H copies
inside the timed region.  ``--impl reference`` times the reference CPU path
(the oracle port, threaded numpy) on the host cores instead.

Unit of ``value``: GB/s of routed rows = Σ_ranks 2·T_l·K·token_bytes (the
rows dispatch delivers plus the rows combine reduces) ÷ step time, whole job.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = json.loads((ROOT / "BASELINE.json").read_text())["metric"] if (ROOT / "BASELINE.json").exists() else \
    "MoE dispatch+combine latency (us) and GB/s/GPU vs NVLink peak, 1-8 B200"

CONFIGS = {
    # name: hidden, dtype, experts, topk, tokens/rank, zipf_s, description
    "oracle": (1024, "f32", 8, 2, 4096, 0.0,
               "synthetic oracle case: hidden 1024 fp32, 8 experts top-2, 4096 tokens/rank, uniform"),
    "mixtral": (4096, "bf16", 8, 2, 8192, 0.0,
                "Mixtral-8x7B shape: hidden 4096 bf16, 8 experts top-2, 8192 tokens/rank, uniform, EP=N"),
    "qwen3": (2048, "bf16", 128, 8, 4096, 0.0,
              "Qwen3-30B-A3B shape: hidden 2048 bf16, 128 experts top-8, 4096 tokens/rank, EP=N"),
    "dsv3": (7168, "bf16", 256, 8, 4096, 0.0,
             "DeepSeek-V3 shape: hidden 7168 bf16, 256 experts top-8, 4096 tokens/rank, per-rank dedup, EP=N"),
    "dsv3_decode": (7168, "bf16", 256, 8, 128, 0.0,
                    "DeepSeek-V3 decode batch: hidden 7168 bf16, 256 experts top-8, 128 tokens/rank, EP=N"),
    "dsv3_zipf": (7168, "bf16", 256, 8, 4096, 1.2,
                  "DeepSeek-V3 shape under Zipf s=1.2 routing, 4096 tokens/rank, EP=N"),
    # diagnostic: top-1, so dispatch push bytes == combine pull bytes (no dedup, no fan-out)
    "k1": (7168, "bf16", 8, 1, 8192, 0.0, "diagnostic: hidden 7168 bf16, 8 experts top-1, 8192 tokens/rank"),
}
# BASELINE.json configs[4]: the 1-8 GPU sweep config, and the largest one that
# BASELINE.json defines at one GPU (the driver's N=1 line and its SCALE sweep)
DEFAULT_CONFIG = "dsv3_zipf"

NVLINK_NOMINAL = 900.0   # GB/s per direction per GPU (NVLink 5)
NVLINK_MEASURED = 770.0  # GB/s peer copy, B200_PROFILING.md


def pattern_ceiling(T: int, K: int, tb: int, dev) -> float | None:
    """HBM GB/s of the P=1 dispatch's access pattern without its metadata:
    T rows read once, each written to K of T*K rows in a random order
    (fs_probe_scatter).  Scattered 14 KB row writes do not reach the
    sequential copy peak; this is the ceiling the dispatch is judged against
    beside the MEASURED_PEAKS copy figure."""
    try:
        from ctypes import c_void_p

        import torch

        from paper_2512_22036_b200 import _lib

        if tb % 16:
            return None
        lib = _lib.load()
        src = torch.empty(T * tb, dtype=torch.uint8, device=dev).fill_(1)
        dst = torch.empty(T * K * tb, dtype=torch.uint8, device=dev)
        perm = torch.randperm(T * K, device=dev).to(torch.int32)
        st = c_void_p(torch.cuda.current_stream().cuda_stream)
        nbytes = T * tb + T * K * tb
        best = 0.0
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        for ctas in (3 * sms, 6 * sms):
            run = lambda: _lib.check(lib.fs_probe_scatter(dev.index or 0, c_void_p(dst.data_ptr()),
                                                          c_void_p(src.data_ptr()), c_void_p(perm.data_ptr()),
                                                          T, K, tb, ctas, st))
            run()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ts = []
            for _ in range(10):
                ev[0].record()
                run()
                ev[1].record()
                ev[1].synchronize()
                ts.append(ev[0].elapsed_time(ev[1]) * 1e-3)
            best = max(best, nbytes / min(ts) / 1e9)
        del src, dst, perm
        torch.cuda.empty_cache()
        return best
    except Exception:  # informational only: never fails the bench line
        return None


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm": float(d["hbm_gbs"]), "hbm_src": "measured (MEASURED_PEAKS.json)"}
    return {"hbm": 6650.0, "hbm_src": "fallback (B200_PROFILING.md)"}


# ---------------------------------------------------------------------------
# algorithmic bytes (host numpy over the routing metadata)


def traffic(experts: np.ndarray, source: np.ndarray, owner: np.ndarray, P: int, tb: int, T_l: int) -> dict:
    own = owner[experts]
    K = experts.shape[1]
    first = np.ones(own.shape, dtype=bool)
    for k in range(1, K):
        first[:, k] = (own[:, :k] != own[:, k : k + 1]).all(axis=1)
    remote = own != source[:, None]
    send = first & remote
    d_eg = np.bincount(source, weights=send.sum(1), minlength=P) * tb
    d_in = np.bincount(own[send], minlength=P) * tb
    c_eg = np.bincount(own[remote], minlength=P) * tb          # rows pulled out of owner g
    c_in = np.bincount(source, weights=remote.sum(1), minlength=P) * tb
    rows = np.bincount(own.reshape(-1), minlength=P)
    # HBM bytes of each kernel on each rank (reads + writes of payload rows):
    # dispatch reads x, every received row is written once, and each duplicate
    # of a remote token is fanned out from its primary row (one more read);
    # combine reads every row once (at its owner) and writes the outputs.
    local_rows = np.bincount(own[~remote], minlength=P)
    primaries_in = np.bincount(own[send], minlength=P)
    dups = rows - local_rows - primaries_in
    hbm_disp = T_l * tb + rows * tb + dups * tb
    hbm_comb = rows * tb + T_l * tb
    # with owner-side pre-reduction (bf16 rows, fp32 accumulate, K <= 8): a
    # token's group of m >= 3 rows on one remote owner crosses as one fp32
    # partial (2 tb) instead of m rows -- the bytes the combine actually pulls
    c_eg_red = np.zeros(P)
    c_in_red = np.zeros(P)
    for g in range(P):
        m = (own == g).sum(1)  # rows of each token on owner g
        rem = source != g
        b = np.where(m >= 3, 2 * tb, m * tb) * rem
        c_eg_red[g] = b.sum()
        c_in_red += np.bincount(source, weights=b, minlength=P)
    return dict(d_eg=d_eg, d_in=d_in, c_eg=c_eg, c_in=c_in, rows=rows, hbm_disp=hbm_disp, hbm_comb=hbm_comb,
                c_eg_red=c_eg_red, c_in_red=c_in_red)


# ---------------------------------------------------------------------------
# clocks


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-i", str(index),
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None

    def stop(self) -> dict | None:
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------


def parse():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="fusco", choices=["fusco", "reference", "nccl"],
                    help="fusco (this repo), reference (CPU oracle port), nccl (disaggregated GPU baseline)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--soak-s", type=float, default=1.5, help="untimed load before timing (clock ramp, sampling)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--graph", action="store_true", default=True,
                    help="time K steps as CUDA-graph replays (default; per-kernel split from an eager pass)")
    ap.add_argument("--eager", dest="graph", action="store_false", help="time K eager launches instead")
    ap.add_argument("--dispatch", choices=["warp", "tma", "auto"], default=os.environ.get("FUSCO_DISPATCH", "auto"),
                    help="dispatch data mover: warp LDG/STG loop or TMA bulk copies")
    ap.add_argument("--combine", choices=["warp", "tma", "auto"], default=os.environ.get("FUSCO_COMBINE", "auto"),
                    help="combine data mover: warp LDG loop or TMA bulk loads into smem stages")
    return ap.parse_args()


def routing_for(cfg_name: str, P: int, seed: int):
    from paper_2512_22036_b200 import box, gen_realworld, round_robin_placement

    hidden, dtype, E, K, T_l, zipf, desc = CONFIGS[cfg_name]
    topo = box(P)
    pl = round_robin_placement(E, topo)
    a = gen_realworld(P * T_l, K, topo, pl, seed=seed, zipf_s=zipf)
    return a, pl


def config_dict(cfg_name: str, P: int, rows_max: int | None = None, nset: int = 2) -> dict:
    """The ``config`` object of the JSON line — identical for both arms."""
    hidden, dtype, E, K, T_l, zipf, desc = CONFIGS[cfg_name]
    tb = hidden * (2 if dtype == "bf16" else 4)
    cfg = {
        "workload": desc,
        "name": cfg_name,
        "ep": P,
        "tokens_per_rank": T_l,
        "hidden": hidden,
        "experts": E,
        "topk": K,
        "zipf_s": zipf,
        "expert": "identity (combine pulls the dispatched rows)",
        "combine_accumulate": "fp32",
        "value_def": "routed-row bytes (dispatch + combine, all ranks) / step time",
    }
    if rows_max is not None:
        cfg["l2"] = (f"inputs larger than L2: {nset} rotating input/output sets + the activation buffer, "
                     f"{(T_l * tb * 2 + rows_max * tb) / 2**20:.0f} MiB touched per step per rank")
    return cfg


def cpu_reference(cfg_name: str, P: int, seed: int, steps: int, warmup: int, budget_s: float = 150.0):
    """Reference CPU path (oracle port) on a bounded sample of the workload."""
    from oracle.cpu_baseline import shuffle_times

    hidden, dtype, E, K, T_l, zipf, desc = CONFIGS[cfg_name]
    a, pl = routing_for(cfg_name, P, seed)
    elem = 2 if dtype == "bf16" else 4
    tb = hidden * elem
    rng = np.random.default_rng(seed + 1)
    T = a.num_tokens

    def run(n_tok):
        sel = np.arange(n_tok)  # first n_tok global tokens: a balanced slice of every rank
        pay = rng.integers(0, 256, size=(n_tok, tb), dtype=np.uint8)
        if dtype == "bf16":  # keep values finite: random sign/exponent-safe bf16 bit patterns
            pay.view(np.uint16)[:] = (pay.view(np.uint16) & 0x3FFF) | 0x3000
        else:
            pay.view(np.float32)[:] = rng.standard_normal((n_tok, tb // 4)).astype(np.float32)
        t = shuffle_times(a.experts[sel], a.weights[sel], a.source[sel], pl.owner, P, pay, dtype)
        return t, 2 * n_tok * K * tb

    # calibrate the sample so warmup+steps fit the budget
    n = min(T, 256)
    (tp, td, tc, thr), _ = run(n)
    per_tok = max((tp + td + tc) / n, 1e-7)
    n = int(min(T, max(64, budget_s / max(1, steps + warmup) / per_tok)))
    vals, lat = [], []
    for i in range(warmup + steps):
        (tp, td, tc, thr), nbytes = run(n)
        if i >= warmup:
            vals.append(nbytes / (tp + td + tc) / 1e9)
            lat.append(tp + td + tc)
    return {
        "value": float(np.median(vals)),
        "unit": "GB/s",
        "cores": int(thr),
        "kind": "port",
        "sample": f"{n} of {T} tokens of the same routing (first {n} global ids, all {P} ranks), "
                  f"plan+dispatch+combine, median of {steps} runs; host os.cpu_count()={os.cpu_count()}",
        "latency_s": float(np.median(lat)),
    }


def run_nccl_baseline(args, world, rank, local, dev) -> int:
    """Disaggregated pack / NCCL all-to-all / unpack on the same config (§8f #1)."""
    import torch
    import torch.distributed as dist

    from paper_2512_22036_b200.baseline import DisaggregatedShuffle

    hidden, dtype, E, K, T_l, zipf, desc = CONFIGS[args.config]
    a, pl = routing_for(args.config, world, args.seed)
    ids = np.flatnonzero(a.source == rank)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    tb = hidden * (2 if dtype == "bf16" else 4)
    x = torch.randn(T_l, hidden, device=dev).to(tdt)
    idx = torch.as_tensor(a.experts[ids], device=dev)
    w = torch.as_tensor(a.weights[ids], dtype=torch.float32, device=dev)
    base = DisaggregatedShuffle(num_experts=E, topk=K, device=dev)

    def step():
        act, st = base.dispatch(x, idx)
        return base.combine(act, st, w)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(args.steps):
        step()
    s1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([s0.elapsed_time(s1) / args.steps], device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    routed = 2.0 * world * T_l * K * tb
    line = {"impl": "nccl", "metric": METRIC, "value": routed / (ms * 1e-3) / 1e9, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "latency_us": ms * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            "config": {"workload": desc, "ep": world},
            "rearrange_bytes_per_rank": DisaggregatedShuffle.rearrange_bytes(T_l, K, tb)}
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def main() -> int:
    args = parse()
    wd = float(os.environ.get("FUSCO_BENCH_WATCHDOG_S", "0"))
    if wd > 0:  # diagnostics: dump every thread's stack and exit if the run hangs
        import faulthandler

        faulthandler.dump_traceback_later(wd, exit=True)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        args.gpus = world
    hidden, dtype, E, K, T_l, zipf, desc = CONFIGS[args.config]

    if args.impl == "reference":
        if rank != 0:
            return 0
        cb = cpu_reference(args.config, world, args.seed, args.steps, args.warmup)
        a_, pl_ = routing_for(args.config, world, args.seed)
        tr_ = traffic(a_.experts, a_.source, pl_.owner, world, hidden * (2 if dtype == "bf16" else 4), T_l)
        line = {
            "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": cb["unit"], "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["latency_s"] * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dtype,
            "data": "synthetic", "config": config_dict(args.config, world, int(tr_["rows"].max())),
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": cb["value"], "unit": cb["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return 0

    import torch
    import torch.distributed as dist

    from paper_2512_22036_b200 import EPBuffer

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if args.impl == "nccl":
        return run_nccl_baseline(args, world, rank, local, dev)
    P = world
    a, pl = routing_for(args.config, P, args.seed)
    elem = 2 if dtype == "bf16" else 4
    tb = hidden * elem
    tr = traffic(a.experts, a.source, pl.owner, P, tb, T_l)
    ids = np.flatnonzero(a.source == rank)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32

    os.environ["FUSCO_DISPATCH"] = args.dispatch
    os.environ["FUSCO_COMBINE"] = args.combine
    buf = EPBuffer(num_experts=E, topk=K, hidden=hidden, dtype=dtype, max_tokens=T_l, with_act_out=False)
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    NSET = 2  # rotate input/output sets so consecutive steps touch different memory (L2 126 MB)
    xs = [torch.randn(T_l, hidden, device=dev, generator=gen).to(tdt) for _ in range(NSET)]
    outs = [torch.empty(T_l, hidden, device=dev, dtype=tdt) for _ in range(NSET)]
    idx = torch.as_tensor(a.experts[ids], device=dev).contiguous()
    w = torch.as_tensor(a.weights[ids], dtype=torch.float32, device=dev).contiguous()
    plan = buf.r.new_plan(idx, with_masks=False)
    r = buf.r
    from ctypes import c_void_p

    from paper_2512_22036_b200 import _lib
    from paper_2512_22036_b200._lib import FS_PHASE_ALL, FS_SRC_ACT

    # Pre-bound C-ABI calls: the timed loop measures the device path, not
    # Python argument marshalling (the e2e number goes through the public API).
    lib = _lib.load()
    stream = c_void_p(torch.cuda.current_stream().cuda_stream)
    h = r.handle
    P_ = lambda t: c_void_p(t.data_ptr())  # noqa: E731
    lay_args = (h, P_(idx), idx.element_size(), T_l, P_(plan.row_of), P_(plan.expert_counts),
                P_(plan.expert_offsets), None, None, P_(plan.stats), FS_PHASE_ALL, stream)
    # dispatch with the router weights: owners pre-reduce a token's groups of
    # >= 3 rows for the fp32-accumulate combine (P > 1; FUSCO_OWNER_REDUCE=0 off)
    disp_args = [(h, P_(xs[j]), P_(idx), idx.element_size(), P_(plan.row_of), P_(w), 4, T_l, FS_PHASE_ALL, stream)
                 for j in range(NSET)]
    comb_args = [(h, P_(idx), idx.element_size(), P_(plan.row_of), P_(w), 4, T_l, P_(outs[j]), buf.dtype_code,
                  FS_SRC_ACT, 0, FS_PHASE_ALL, stream) for j in range(NSET)]
    f_layout, f_disp, f_comb = lib.fs_layout, lib.fs_dispatch_w, lib.fs_combine

    def step(j, ev=None):
        if ev is not None:
            ev[0].record()
        rc = f_layout(*lay_args)
        if ev is not None:
            ev[1].record()
        rc |= f_disp(*disp_args[j % NSET])
        if ev is not None:
            ev[2].record()
        rc |= f_comb(*comb_args[j % NSET])
        if ev is not None:
            ev[3].record()
        if rc:
            _lib.check(rc)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # correctness guard before timing (cheap): a round trip must reproduce x (weights sum to 1)
    step(0)
    buf.check()
    plan.epoch = r.epoch
    rt = (xs[0].float() * w.sum(1, keepdim=True)).to(tdt).float()
    if not torch.allclose(outs[0].float(), rt, rtol=2.0**-7, atol=2e-2):
        raise SystemExit("bench: round-trip check failed")

    sampler = ClockSampler(local)
    for i in range(args.warmup):
        step(i)
    barrier()
    t_end = time.time() + args.soak_s
    j = 0
    while time.time() < t_end:
        for _ in range(20):
            step(j)
            j += 1
        torch.cuda.synchronize()
    barrier()

    # ---- timed region: EXACTLY K steps, device time, max over ranks --------
    # Per-kernel CUDA events on the launching stream give each kernel's
    # average duration inside the timed region (roofline).  With --graph the
    # K steps replay a captured 2-step CUDA graph (launch-bound configs); the
    # per-kernel split then comes from an eager pass of the same K steps.
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    graph = None
    if args.graph:
        gs = torch.cuda.Stream()
        gs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(gs):
            graph = torch.cuda.CUDAGraph()
            stream_g = c_void_p(gs.cuda_stream)
            lay_args = lay_args[:-1] + (stream_g,)
            disp_args = [d[:-1] + (stream_g,) for d in disp_args]
            comb_args = [c[:-1] + (stream_g,) for c in comb_args]
            with torch.cuda.graph(graph, stream=gs):
                step(0)
                step(1)
        torch.cuda.current_stream().wait_stream(gs)
        lay_args = lay_args[:-1] + (stream,)
        disp_args = [d[:-1] + (stream,) for d in disp_args]
        comb_args = [c[:-1] + (stream,) for c in comb_args]
        for _ in range(3):
            graph.replay()
    nvc, nvc_err = None, None
    if P > 1:  # NVLink data counters (ncu cannot wrap a multi-rank run)
        try:
            from paper_2512_22036_b200.nvlink import NvlinkCounters

            nvc = NvlinkCounters(dev)
        except Exception as e:  # measurement only: report why it is missing
            nvc, nvc_err = None, repr(e)
    barrier()
    host0 = time.perf_counter()
    start.record()
    if graph is not None:
        for i in range(args.steps // 2):
            graph.replay()
        if args.steps % 2:
            step(args.steps - 1)
    else:
        for i in range(args.steps):
            step(i, evs[i])
    end.record()
    host_ms = (time.perf_counter() - host0) * 1e3
    barrier()
    buf.check()
    total_ms = start.elapsed_time(end)
    link_step = link_disp = None
    n_cnt = max(args.steps, 200)  # counter passes: long enough for the NVML sampling
    if nvc:
        # whole steps, then the same number without the combine (the
        # dispatch's and planner's own link bytes); outside the timed region
        nvc.start()
        for i in range(n_cnt):
            step(i)
        barrier()
        link_step = nvc.stop()
        for i in range(n_cnt):
            f_layout(*lay_args)
            f_disp(*disp_args[i % NSET])
        barrier()
        nvc.start()
        for i in range(n_cnt):
            f_layout(*lay_args)
            f_disp(*disp_args[i % NSET])
        barrier()
        link_disp = nvc.stop()
        buf.check()
    if graph is not None:  # per-kernel split from an eager pass of the same K steps
        barrier()
        for i in range(args.steps):
            step(i, evs[i])
        barrier()
    k_layout = sum(e[0].elapsed_time(e[1]) for e in evs) / args.steps
    k_disp = sum(e[1].elapsed_time(e[2]) for e in evs) / args.steps
    k_comb = sum(e[2].elapsed_time(e[3]) for e in evs) / args.steps
    launches = 3 * args.steps

    # ---- e2e: public API, pinned host buffers, copies inside the timed region.
    # Every step copies its inputs H2D and its output D2H; steps are pipelined
    # over three streams (H2D of step j+1 and D2H of step j-1 overlap step j's
    # shuffle — PCIe is full duplex), the way a serving loop would run it.
    e2e = None
    if not args.no_e2e:
        xh = [x.cpu().pin_memory() for x in xs]
        oh = [torch.empty(T_l, hidden, dtype=tdt).pin_memory() for _ in range(NSET)]
        idx_h = torch.as_tensor(a.experts[ids]).pin_memory()
        w_h = torch.as_tensor(a.weights[ids], dtype=torch.float32).pin_memory()
        xd = [torch.empty_like(xs[0]) for _ in range(NSET)]
        idx_d = [torch.empty_like(idx) for _ in range(NSET)]
        w_d = [torch.empty_like(w) for _ in range(NSET)]
        od = [torch.empty_like(xs[0]) for _ in range(NSET)]
        s_in, s_cmp, s_out = torch.cuda.Stream(), torch.cuda.current_stream(), torch.cuda.Stream()
        ev_in = [torch.cuda.Event() for _ in range(NSET)]     # inputs of slot landed
        ev_used = [torch.cuda.Event() for _ in range(NSET)]   # shuffle done reading slot inputs
        ev_done = [torch.cuda.Event() for _ in range(NSET)]   # output of slot computed
        ev_out = [torch.cuda.Event() for _ in range(NSET)]    # output of slot copied out
        for e_ in ev_used + ev_out:
            e_.record(s_cmp)

        def e2e_step(j):
            q = j % NSET
            with torch.cuda.stream(s_in):
                s_in.wait_event(ev_used[q])
                xd[q].copy_(xh[q], non_blocking=True)
                idx_d[q].copy_(idx_h, non_blocking=True)
                w_d[q].copy_(w_h, non_blocking=True)
                ev_in[q].record(s_in)
            s_cmp.wait_event(ev_in[q])
            s_cmp.wait_event(ev_out[q])
            p = buf.build_plan(idx_d[q], stream=s_cmp)
            buf.dispatch(xd[q], p, stream=s_cmp, topk_w=w_d[q])
            buf.combine(p, w_d[q], out=od[q], src="act", stream=s_cmp)
            ev_used[q].record(s_cmp)
            ev_done[q].record(s_cmp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_done[q])
                oh[q].copy_(od[q], non_blocking=True)
                ev_out[q].record(s_out)

        def drain():
            s_cmp.wait_stream(s_in)
            s_cmp.wait_stream(s_out)

        for i in range(max(3, args.warmup // 4)):
            e2e_step(i)
        drain()
        barrier()
        s2, t2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s2.record(s_cmp)
        s_in.wait_event(s2)
        s_out.wait_event(s2)
        for i in range(args.steps):
            e2e_step(i)
        drain()
        t2.record(s_cmp)
        barrier()
        e2e_ms = s2.elapsed_time(t2)
        h2d = T_l * tb + T_l * K * 8 + T_l * K * 4
        e2e = {"ms": e2e_ms, "h2d": h2d, "d2h": T_l * tb}
    clocks = sampler.stop()

    vec = torch.tensor([total_ms, k_layout, k_disp, k_comb, e2e["ms"] if e2e else 0.0], dtype=torch.float64,
                       device=dev)
    links = None
    if world > 1:
        dist.all_reduce(vec, op=dist.ReduceOp.MAX)
        lk = torch.tensor([float(link_step[0]), float(link_step[1]), float(link_disp[0]), float(link_disp[1])]
                          if nvc else [-1.0] * 4, dtype=torch.float64, device=dev)
        allk = [torch.empty_like(lk) for _ in range(world)]
        dist.all_gather(allk, lk)
        links = torch.stack(allk).cpu().numpy() / n_cnt  # [P, 4] bytes per step
    total_ms, k_layout, k_disp, k_comb, e2e_ms = vec.tolist()
    ms = total_ms / args.steps
    routed = 2.0 * P * T_l * K * tb  # bytes per step, whole job
    value = routed / (ms * 1e-3) / 1e9

    # the library's default for owner pre-reduction (fs_combine), reported on the line
    owner_reduce = bool(P > 1 and (3 if dtype == "bf16" else 2) <= K <= 8 and args.combine in ("auto", "tma")
                        and os.environ.get("FUSCO_OWNER_REDUCE") != "0"
                        and (os.environ.get("FUSCO_OWNER_REDUCE") == "1"
                             or (T_l > 512 and (P == 2 or (P <= 4 and tb >= 8192)))))
    pk = peaks()
    if P == 1:
        disp_b, comb_b = float(tr["hbm_disp"][0]), float(tr["hbm_comb"][0])
        t_min_d, t_min_c = disp_b / (pk["hbm"] * 1e9), comb_b / (pk["hbm"] * 1e9)
        dom = "fs_dispatch" if k_disp >= k_comb else "fs_combine"
        b, t = (disp_b, k_disp) if dom == "fs_dispatch" else (comb_b, k_comb)
        achieved = b / (t * 1e-3) / 1e9
        roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": pk["hbm"], "unit": "GB/s",
                "frac": achieved / pk["hbm"], "peak_src": pk["hbm_src"], "bytes_per_launch": b,
                "traffic": None}
        if dom == "fs_dispatch":
            pc = pattern_ceiling(T_l, K, tb, dev)
            if pc:
                roof["pattern_ceiling"] = {"value": pc, "unit": "GB/s", "frac": achieved / pc,
                                           "src": "fs_probe_scatter in-run: the same rows read once and written "
                                                  "to K scattered rows with plain 16-byte stores, no metadata "
                                                  "(best of 2 grids, 10 reps)"}
    else:
        # bottleneck rank's NVLink bytes (max of egress / ingress over ranks);
        # the kernel floor is the slower of that over the link and its HBM bytes
        d_bn = float(np.maximum(tr["d_eg"], tr["d_in"]).max())
        c_bn = float(np.maximum(tr["c_eg"], tr["c_in"]).max())
        t_min_d = max(d_bn / (NVLINK_NOMINAL * 1e9), float(tr["hbm_disp"].max()) / (pk["hbm"] * 1e9))
        t_min_c = max(c_bn / (NVLINK_NOMINAL * 1e9), float(tr["hbm_comb"].max()) / (pk["hbm"] * 1e9))
        dom = "fs_dispatch" if k_disp >= k_comb else "fs_combine"
        b, t = (d_bn, k_disp) if dom == "fs_dispatch" else (c_bn, k_comb)
        achieved = b / (t * 1e-3) / 1e9
        roof = {"bound": "nvlink", "kernel": dom, "achieved": achieved, "peak": NVLINK_MEASURED, "unit": "GB/s",
                "frac": achieved / NVLINK_MEASURED, "peak_src": "measured peer copy 770 GB/s/dir (B200_PROFILING.md)",
                "frac_of_nominal_900": achieved / NVLINK_NOMINAL,
                "bytes_per_launch": b, "traffic": None}
        if dom == "fs_combine" and owner_reduce:
            # the bytes this combine actually moves (owner pre-reduction): the
            # link's physical utilisation beside the reference-bytes figure
            lb = float(np.maximum(tr["c_eg_red"], tr["c_in_red"]).max())
            roof["link_bytes_per_launch"] = lb
            roof["link_achieved"] = lb / (t * 1e-3) / 1e9
            roof["link_frac"] = roof["link_achieved"] / NVLINK_MEASURED
    traffic_file = ROOT / "profiles" / "ncu_traffic.json"
    if traffic_file.exists() and P == 1:
        tf = json.loads(traffic_file.read_text())
        roof["traffic"] = tf.get(f"{args.config}/n{P}/{dom}")
    nvl_file = ROOT / "profiles" / f"r2_nvl_counters_{args.config}_ep{P}.json"
    if P > 1 and nvl_file.exists():
        # ncu counters of the same kernel on P real GPUs (tools/ncu_nvlink.py, phased
        # run): DRAM bytes per launch and the NVLink bytes it moved (push TX / pull RX)
        try:
            ks = [k for k in json.loads(nvl_file.read_text())["kernels"]
                  if k["kernel"] == dom and k["phase"] == ("local" if dom == "fs_dispatch" else "remote")]
            if ks:
                roof["traffic"] = float(np.mean([k["dram_bytes"] for k in ks]))
                roof["nvlink_counter_bytes"] = float(np.max([k["nvl_tx_bytes" if dom == "fs_dispatch"
                                                               else "nvl_rx_bytes"] for k in ks]))
                roof["counters_src"] = f"profiles/{nvl_file.name} (ncu, owner pre-reduction as in that run)"
        except (OSError, KeyError, ValueError):
            pass
    nvlink = None
    if links is not None and (links >= 0).all():
        # measured link bytes per step and GPU against the algorithmic bytes
        # (push: source TX / owner RX; pull: owner TX / puller RX)
        disp_tx, disp_rx = links[:, 2], links[:, 3]
        comb_tx, comb_rx = links[:, 0] - disp_tx, links[:, 1] - disp_rx
        per = []
        for g in range(P):
            per.append({"gpu": g, "dispatch_tx": disp_tx[g], "dispatch_rx": disp_rx[g],
                        "alg_dispatch_tx": float(tr["d_eg"][g]), "alg_dispatch_rx": float(tr["d_in"][g]),
                        "combine_tx": comb_tx[g], "combine_rx": comb_rx[g],
                        "alg_combine_tx": float(tr["c_eg"][g]), "alg_combine_rx": float(tr["c_in"][g])})
        meas = {"fs_dispatch": float(np.maximum(disp_tx, disp_rx).max()),
                "fs_combine": float(np.maximum(comb_tx, comb_rx).max())}
        nvlink = {
            "source": f"NVML NVLink data counters ({nvc.mode if nvc else 'n/a'}) over {n_cnt} steps after the "
                      "timed region; dispatch from a layout+dispatch-only pass of as many steps, combine = step - "
                      "dispatch",
            "per_gpu_bytes_per_step": [{k: (round(float(v)) if k != "gpu" else v) for k, v in d.items()} for d in per],
            "bottleneck_bytes": {"fs_dispatch": {"measured": meas["fs_dispatch"], "algorithmic": d_bn},
                                 "fs_combine": {"measured": meas["fs_combine"], "algorithmic": c_bn}},
            "measured_over_algorithmic": {k: meas[k] / ((d_bn if k == "fs_dispatch" else c_bn) or 1.0)
                                          for k in meas},
            "gbps_per_gpu_measured": {"fs_dispatch": meas["fs_dispatch"] / (k_disp * 1e-3) / 1e9,
                                      "fs_combine": meas["fs_combine"] / (k_comb * 1e-3) / 1e9},
        }
        roof["traffic"] = meas[dom]
        roof["traffic_src"] = "NVLink data bytes of the bottleneck GPU per launch (NVML counters)"
    elif P > 1:
        nvlink = {"unavailable": nvc_err or "counters not readable on every rank"}

    line = {
        "metric": METRIC,
        "value": value,
        "unit": "GB/s",
        "n_gpus": P,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": dtype,
        "data": "synthetic: reference gen_realworld routing (seed 0) + random payload rows",
        "config": config_dict(args.config, P, int(tr["rows"].max()), NSET),
        "latency_us": ms * 1e3,
        "kernel_us": {"fs_layout": k_layout * 1e3, "fs_dispatch": k_disp * 1e3, "fs_combine": k_comb * 1e3},
        "t_min_us": {"fs_dispatch": t_min_d * 1e6, "fs_combine": t_min_c * 1e6},
        "roofline_step_frac": (t_min_d + t_min_c) / (ms * 1e-3),
        "nvlink_gbps_per_gpu": None if P == 1 else {
            "dispatch": float(tr["d_eg"].mean()) / (k_disp * 1e-3) / 1e9,
            "combine": float(tr["c_eg"].mean()) / (k_comb * 1e-3) / 1e9,
        },
        # combine bytes that actually cross NVLink when owners pre-reduce
        # (the algorithmic "combine" above counts every remote (t, k) row)
        "combine_link_bytes_per_gpu": None if P == 1 else {
            "algorithmic_rows": float(tr["c_eg"].mean()), "pulled_with_owner_reduce": float(tr["c_eg_red"].mean()),
            "link_gbps_with_owner_reduce": float(tr["c_eg_red"].mean()) / (k_comb * 1e-3) / 1e9,
        },
        "gbps_per_gpu": value / P,
        "roofline": roof,
        "nvlink_counters": nvlink,
        "gpu_launches": launches,
        "launch_mode": "cuda_graph" if graph is not None else "eager",
        "dispatch_engine": args.dispatch if args.dispatch != "auto" else ("tma" if P == 1 else "warp"),
        "combine_engine": args.combine if args.combine != "auto" else ("warp" if P == 1 else "tma"),
        "owner_reduce": owner_reduce,
        "host_enqueue_ms_per_step": host_ms / args.steps,
        "clocks": clocks,
    }
    if e2e is not None:
        line["e2e"] = {"value": routed / (e2e_ms / args.steps * 1e-3) / 1e9, "unit": "GB/s",
                       "ms_per_step": e2e_ms / args.steps, "h2d_bytes_per_step": e2e["h2d"] * P,
                       "d2h_bytes_per_step": e2e["d2h"] * P,
                       "pipeline": "3 streams: H2D(j+1) | shuffle(j) | D2H(j-1), pinned host buffers"}
    if rank == 0 and not args.no_cpu_baseline:
        cb = cpu_reference(args.config, world, args.seed, steps=3, warmup=1, budget_s=25.0)
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
    buf.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
