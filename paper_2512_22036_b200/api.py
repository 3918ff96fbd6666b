"""Reference-shaped entry points, executed on the GPU.

Same names, argument meaning and error behaviour as the reference package
(``shuffleforge``), so its callers and tests switch over unchanged:

* ``run_exchange``   — reference engine.py:374-460: plan + dispatch + expert
  function + combine for a whole (emulated) cluster in one process.  Here all
  P ranks run on the current GPU through the NVLink kernels (see
  ``engine.EmulatedCluster``).  Results are bit-identical to the reference:
  activations byte-for-byte, outputs bit-for-bit with ``acc="f64"``
  (the default, the reference's f64 k-ascending reduction).
* ``build_plan_pair`` — reference planner.py:485-497, planned on device.
* ``dispatch_loads`` / ``dedup_ratio`` — reference planner.py:178-208,
  662-673, from the device planner's counters.

Payloads follow the reference: float32 rows (``make_token_payloads``,
engine.py:238-246); ``dtype="bf16"`` interprets the same byte rows as bf16.
Expert functions take and return torch tensors on the device.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import balancer as _balancer
from .engine import EmulatedCluster, Plan, dtype_code, _ACCS
from ._lib import FS_SRC_ACT, FS_SRC_ACT_OUT, STAT_NAIVE_SEND, STAT_NODE_DEDUP, STAT_LOCAL_ROWS
from .routing import RoutingAssignment
from .topology import ClusterTopology, ExpertPlacement

ABLATIONS = ("dcomm", "planner", "balancer")


def make_token_payloads(num_tokens: int, token_bytes: int, seed: int) -> np.ndarray:
    """float32 standard-normal rows as bytes (reference engine.py:238-246)."""
    if token_bytes % 4:
        raise ValueError("token_bytes must be a multiple of 4 (float32 payloads)")
    vals = np.random.default_rng(seed).standard_normal((num_tokens, token_bytes // 4)).astype(np.float32)
    return vals.view(np.uint8).reshape(num_tokens, token_bytes)


def identity_expert(activations: torch.Tensor, expert_ids: torch.Tensor) -> torch.Tensor:
    return activations


def scaled_expert(num_experts: int):
    """Expert e computes x*(e+2)+e in float32 (reference engine.py:283-292)."""

    def fn(activations: torch.Tensor, expert_ids: torch.Tensor) -> torch.Tensor:
        e = expert_ids.to(torch.float32)[:, None]
        return activations * (e + 2) + e

    return fn


@dataclass(frozen=True)
class ActivationLayout:
    """Provenance of every activation row of one rank (planner.py:89-104)."""

    expert_ids: np.ndarray = field(repr=False)
    token_ids: np.ndarray = field(repr=False)
    src_flat: np.ndarray = field(repr=False)
    k_col: np.ndarray = field(repr=False)

    @property
    def num_rows(self) -> int:
        return int(self.token_ids.size)


@dataclass
class GpuPlan:
    """Host view of the device plan (the reference's CommPlan fields that
    survive without descriptor lists: the row layout is the plan)."""

    direction: str
    token_bytes: int
    num_tokens: int
    topk: int
    groups: np.ndarray | None
    layouts: dict[int, ActivationLayout]
    local_tokens: dict[int, np.ndarray]
    row_of: np.ndarray           # [T, K] global
    first_mask: np.ndarray       # [T, K] token-node first appearance
    reduce_weights: dict[int, np.ndarray] | None
    inter_bytes_total: int
    intra_bytes_total: int
    intra_gpu_bytes: int
    buffer_bytes: dict[str, int]
    loads: np.ndarray            # per-rank dedup send bytes (dispatch_loads)


@dataclass
class PhaseReport:
    """Measured (CUDA events) stage times and byte counters of one direction
    (reference engine.py:60-90; ``rearrange`` is structurally zero: there is
    no standalone permute pass)."""

    direction: str
    mode: str
    preprocess_s: float
    rearrange_s: float
    communicate_s: float
    inter_node_bytes: int
    intra_node_bytes: int
    intra_gpu_bytes: int
    rearrange_bytes: int

    @property
    def total_s(self) -> float:
        return self.preprocess_s + self.rearrange_s + self.communicate_s

    def to_json(self) -> dict:
        return {
            "direction": self.direction,
            "mode": self.mode,
            "preprocess_s": self.preprocess_s,
            "rearrange_s": self.rearrange_s,
            "communicate_s": self.communicate_s,
            "total_s": self.total_s,
            "inter_node_bytes": self.inter_node_bytes,
            "intra_node_bytes": self.intra_node_bytes,
            "intra_gpu_bytes": self.intra_gpu_bytes,
            "rearrange_bytes": self.rearrange_bytes,
        }


@dataclass
class ExchangeResult:
    mode: str
    groups: np.ndarray | None
    dispatch_plan: GpuPlan
    combine_plan: GpuPlan
    dispatch_report: PhaseReport
    combine_report: PhaseReport
    payloads: np.ndarray | None
    buffers: dict[str, np.ndarray] | None

    def _buf(self, kind: str, g: int) -> np.ndarray:
        if self.buffers is None:
            raise ValueError("run was not materialized; no buffer contents")
        return self.buffers[f"{kind}/{g}"]

    def activation(self, g: int) -> np.ndarray:
        return self._buf("activation", g)

    def output(self, s: int) -> np.ndarray:
        return self._buf("output", s)

    def output_f32(self, s: int) -> np.ndarray:
        return self.output(s).view(np.float32).reshape(-1, self.combine_plan.token_bytes // 4)

    @property
    def total_s(self) -> float:
        return self.dispatch_report.total_s + self.combine_report.total_s


# ---------------------------------------------------------------------------


def _validate(assignment, topo, placement, token_bytes, mode="analytic", ablate=()):
    ablate = frozenset(ablate)
    unknown = ablate - set(ABLATIONS)
    if unknown:
        raise ValueError(f"unknown ablations: {sorted(unknown)}")
    if mode not in ("analytic", "wallclock"):
        raise ValueError(f"unknown mode {mode!r}")
    if mode == "wallclock" and "dcomm" in ablate:
        raise ValueError("the dcomm ablation redefines the cost model only; meaningless in wallclock mode")
    if token_bytes % 4 or token_bytes <= 0:
        raise ValueError("token_bytes must be a positive multiple of 4")
    assignment.validate(topo, placement)
    placement.validate(topo)
    if topo.num_gpus > 32:
        raise ValueError("at most 32 ranks per shuffle (one NVSwitch domain)")
    return ablate


class _Session:
    """Routing of a global assignment split into per-rank device tensors."""

    def __init__(self, assignment, topo, placement, token_bytes, *, with_act_out, device=None, nodedup=False):
        self.P = topo.num_gpus
        self.a = assignment
        self.topo = topo
        self.placement = placement
        self.tb = token_bytes
        self.dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.ids = [np.flatnonzero(assignment.source == s) for s in range(self.P)]
        max_t = max([i.size for i in self.ids] + [1])
        self.cluster = EmulatedCluster(
            self.P, placement.num_experts, assignment.topk, token_bytes, max_t,
            owner=placement.owner, node_of=topo.node_table(), with_act_out=with_act_out, device=self.dev,
            nodedup=nodedup,
        )
        self.idx = [torch.as_tensor(assignment.experts[i], dtype=torch.int64, device=self.dev).contiguous()
                    for i in self.ids]

    def close(self):
        self.cluster.close()

    def plans(self) -> list[Plan]:
        return self.cluster.layout(self.idx, with_masks=True)

    def host_plan(self, plans: list[Plan], direction: str, groups) -> GpuPlan:
        a, P, tb, K = self.a, self.P, self.tb, self.a.topk
        owner = self.placement.owner
        row_of = np.full((a.num_tokens, K), -1, dtype=np.int64)
        first = np.zeros((a.num_tokens, K), dtype=bool)
        stats = np.zeros((P, 8), dtype=np.int64)
        for s, p in enumerate(plans):
            row_of[self.ids[s]] = p.row_of.cpu().numpy()
            first[self.ids[s]] = p.first_mask.cpu().numpy().astype(bool)
            stats[s] = p.stats.cpu().numpy()
        rows = [int(p.expert_offsets[-1].item()) for p in plans]
        layouts = {}
        own = owner[a.experts]
        for g in range(P):
            ts, ks = np.nonzero(own == g)
            r = row_of[ts, ks]
            e_ids = np.empty(rows[g], dtype=np.int64)
            t_ids = np.empty(rows[g], dtype=np.int64)
            k_col = np.empty(rows[g], dtype=np.int64)
            e_ids[r], t_ids[r], k_col[r] = a.experts[ts, ks], ts, ks
            layouts[g] = ActivationLayout(e_ids, t_ids, a.source[t_ids], k_col)
        m = self.topo.gpus_per_node
        loads = stats[:, STAT_NODE_DEDUP] * tb
        same_gpu = int(stats[:, STAT_LOCAL_ROWS].sum()) * tb
        naive_rows = 0
        for s in range(P):  # same-node, other-GPU rows (intra-node traffic)
            g = own[self.ids[s]]
            naive_rows += int(((g // m == s // m) & (g != s)).sum())
        if direction == "dispatch":
            inter = int(loads.sum())
            buffer_bytes = {**{f"token/{s}": self.ids[s].size * tb for s in range(P)},
                            **{f"activation/{g}": rows[g] * tb for g in range(P)}}
            reduce_w = None
        else:
            inter = int(sum(int((own[self.ids[s]] // m != s // m).sum()) for s in range(P))) * tb
            buffer_bytes = {**{f"act_out/{g}": rows[g] * tb for g in range(P)},
                            **{f"output/{s}": self.ids[s].size * tb for s in range(P)}}
            reduce_w = {s: a.weights[self.ids[s]] for s in range(P)}
        return GpuPlan(
            direction=direction, token_bytes=tb, num_tokens=a.num_tokens, topk=K, groups=groups,
            layouts=layouts, local_tokens={s: self.ids[s] for s in range(P)}, row_of=row_of,
            first_mask=first, reduce_weights=reduce_w, inter_bytes_total=inter,
            intra_bytes_total=naive_rows * tb, intra_gpu_bytes=same_gpu, buffer_bytes=buffer_bytes,
            loads=loads,
        )


def _open_session(assignment, topo, placement, token_bytes, ablate, *, with_act_out, device=None) -> _Session:
    """A session whose ranks push without dedup when ``planner`` is ablated
    (every (token, k) row crosses the link, ``fs_set_nodedup``)."""
    return _Session(assignment, topo, placement, token_bytes, with_act_out=with_act_out, device=device,
                    nodedup="planner" in ablate)


def build_plan_pair(
    assignment: RoutingAssignment,
    topo: ClusterTopology,
    placement: ExpertPlacement,
    token_bytes: int,
    balancer: str = "greedy",
    device=None,
) -> tuple[GpuPlan, GpuPlan, np.ndarray]:
    """Device-planned (dispatch, combine, groups) (reference planner.py:485-497)."""
    _validate(assignment, topo, placement, token_bytes)
    sess = _Session(assignment, topo, placement, token_bytes, with_act_out=False, device=device)
    try:
        plans = sess.plans()
        sess.cluster.check()
        d = sess.host_plan(plans, "dispatch", None)
        groups = _balancer.build_groups(balancer, d.loads, topo)
        d.groups = groups
        c = sess.host_plan(plans, "combine", groups)
        return d, c, groups
    finally:
        sess.close()


# SPEC.md:260 name
def build_plan(assignment, placement, topology, groups=None, token_bytes: int = 4, device=None) -> GpuPlan:
    d, _, g = build_plan_pair(assignment, topology, placement, token_bytes, device=device)
    if groups is not None:
        _balancer.validate_groups(groups, topology)
        d.groups = np.asarray(groups)
    return d


def dispatch_loads(assignment, placement, topo, token_bytes, device=None) -> np.ndarray:
    """Per-rank deduplicated remote send bytes (reference planner.py:178-196)."""
    d, _, _ = build_plan_pair(assignment, topo, placement, token_bytes, device=device)
    return d.loads


def naive_inter_node_bytes(assignment, placement, topo, token_bytes) -> int:
    m = topo.gpus_per_node
    return int((placement.owner[assignment.experts] // m != (assignment.source // m)[:, None]).sum()) * token_bytes


def dedup_ratio(assignment, topo, placement, device=None) -> float:
    naive = naive_inter_node_bytes(assignment, placement, topo, 1)
    dedup = int(dispatch_loads(assignment, placement, topo, 4, device=device).sum()) // 4
    if dedup == 0:
        return 1.0 if naive == 0 else float("inf")
    return naive / dedup


def run_exchange(
    assignment: RoutingAssignment,
    topo: ClusterTopology,
    placement: ExpertPlacement,
    token_bytes: int,
    *,
    payload_seed: int = 0,
    balancer: str = "greedy",
    mode: str = "analytic",
    cost=None,
    ablate=(),
    expert_fn=identity_expert,
    materialize: bool = True,
    dtype: str = "f32",
    acc: str = "f64",
    device=None,
) -> ExchangeResult:
    """Plan, dispatch, run experts, combine — on the GPU (reference engine.py:374-460).

    ``mode``/``cost`` are accepted for signature compatibility: both modes
    execute the real kernels and report CUDA-event times.  The ``planner`` and
    ``dcomm`` ablations (no dedup / disaggregated pack-a2a-unpack) are the
    next-row GPU baseline and are not implemented on this path yet.
    """
    ablate = _validate(assignment, topo, placement, token_bytes, mode, ablate)
    tdt, code = dtype_code(dtype)
    if acc not in _ACCS:
        raise ValueError("acc must be 'f32' or 'f64'")
    if "dcomm" in ablate:
        return _run_disaggregated(assignment, topo, placement, token_bytes, payload_seed=payload_seed,
                                  balancer=balancer, mode=mode, expert_fn=expert_fn, materialize=materialize,
                                  dtype=dtype, acc=acc, device=device)
    identity = expert_fn is identity_expert
    sess = _open_session(assignment, topo, placement, token_bytes, ablate, with_act_out=not identity, device=device)
    try:
        cl, P, dev = sess.cluster, sess.P, sess.dev
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        ev[0].record()
        plans = sess.plans()
        ev[1].record()
        payloads = make_token_payloads(assignment.num_tokens, token_bytes, payload_seed)
        xs = [torch.as_tensor(payloads[i], device=dev).contiguous() for i in sess.ids]
        ws = [torch.as_tensor(assignment.weights[i], dtype=torch.float64 if acc == "f64" else torch.float32,
                              device=dev).contiguous() for i in sess.ids]
        outs = [torch.empty((i.size, token_bytes), dtype=torch.uint8, device=dev) for i in sess.ids]
        ev[2].record()
        cl.dispatch(xs, plans)
        ev[3].record()
        rows = [p.num_rows for p in plans]
        if not identity:
            for r, p, n in zip(cl.ranks, plans, rows):
                counts = p.expert_counts.to(torch.int64)
                eids = torch.repeat_interleave(torch.as_tensor(r.local_experts, device=dev), counts)
                act = r.act(n, tdt)
                y = expert_fn(act.to(torch.float32), eids)
                if tuple(y.shape) != tuple(act.shape):
                    raise ValueError("expert function changed the activation shape")
                r.act_out(n, tdt).copy_(y.to(tdt))
        ev[4].record()
        cl.combine(plans, ws, [o.view(tdt) for o in outs], dtype_code=code,
                   src=FS_SRC_ACT if identity else FS_SRC_ACT_OUT, acc=_ACCS[acc])
        ev[5].record()
        cl.check()
        d = sess.host_plan(plans, "dispatch", None)
        groups = _balancer.build_groups(balancer if "balancer" not in ablate else "static", d.loads, topo)
        d.groups = groups
        c = sess.host_plan(plans, "combine", groups)
        buffers = None
        if materialize or mode == "wallclock":
            buffers = {}
            for g, (r, n) in enumerate(zip(cl.ranks, rows)):
                buffers[f"activation/{g}"] = r.act(n).reshape(-1).cpu().numpy()
                buffers[f"output/{g}"] = outs[g].reshape(-1).cpu().numpy()
        t_plan = ev[0].elapsed_time(ev[1]) * 1e-3
        t_disp = ev[2].elapsed_time(ev[3]) * 1e-3
        t_comb = ev[4].elapsed_time(ev[5]) * 1e-3
        if "planner" in ablate:
            d.inter_bytes_total = naive_inter_node_bytes(assignment, placement, topo, token_bytes)
            d.groups = None
            c.groups = None
            groups = None
        drep = PhaseReport("dispatch", mode, t_plan, 0.0, t_disp, d.inter_bytes_total, d.intra_bytes_total,
                           d.intra_gpu_bytes, 0)
        crep = PhaseReport("combine", mode, 0.0, 0.0, t_comb, c.inter_bytes_total, c.intra_bytes_total,
                           c.intra_gpu_bytes, 0)
        return ExchangeResult(mode, groups, d, c, drep, crep, payloads if (materialize or mode == "wallclock") else None,
                              buffers)
    finally:
        sess.close()


def _run_disaggregated(assignment, topo, placement, token_bytes, *, payload_seed, balancer, mode, expert_fn,
                       materialize, dtype, acc, device):
    """ablate={"dcomm"}: the disaggregated pack / all-to-all / unpack shuffle
    (reference run_baseline, engine.py:552-625) with the same output bytes;
    rearrange bytes = 4 passes (engine.py:628-630)."""
    from .baseline import emulated_exchange

    tdt, _ = dtype_code(dtype)
    sess = _Session(assignment, topo, placement, token_bytes, with_act_out=False, device=device)
    try:
        plans = sess.plans()  # layouts / counters for the host plan objects
        sess.cluster.check()
        d = sess.host_plan(plans, "dispatch", None)
        c = sess.host_plan(plans, "combine", None)
    finally:
        sess.close()
    dev = sess.dev
    payloads = make_token_payloads(assignment.num_tokens, token_bytes, payload_seed)
    xs = [torch.as_tensor(payloads[i], device=dev).contiguous().view(tdt) for i in sess.ids]
    idxs = [torch.as_tensor(assignment.experts[i], device=dev) for i in sess.ids]
    ws = [torch.as_tensor(assignment.weights[i], dtype=torch.float64, device=dev) for i in sess.ids]
    fn = None if expert_fn is identity_expert else expert_fn
    acts, outs, ((dr, dc), (cr, cc)) = emulated_exchange(xs, idxs, ws, placement.owner, sess.P, fn, tdt, acc)
    rows = 2 * assignment.num_tokens * assignment.topk * token_bytes  # pack + unpack, per direction
    naive = naive_inter_node_bytes(assignment, placement, topo, token_bytes)
    d.inter_bytes_total = naive
    d.groups = c.groups = None
    drep = PhaseReport("dispatch", mode, 0.0, dr, dc, naive, d.intra_bytes_total, d.intra_gpu_bytes, rows)
    crep = PhaseReport("combine", mode, 0.0, cr, cc, c.inter_bytes_total, c.intra_bytes_total, c.intra_gpu_bytes,
                       rows)
    buffers = None
    if materialize or mode == "wallclock":
        buffers = {}
        for g in range(sess.P):
            buffers[f"activation/{g}"] = acts[g].contiguous().view(torch.uint8).reshape(-1).cpu().numpy()
            buffers[f"output/{g}"] = outs[g].contiguous().view(torch.uint8).reshape(-1).cpu().numpy()
    return ExchangeResult(mode, None, d, c, drep, crep, payloads if buffers is not None else None, buffers)


# SPEC.md:396,405 names for the whole-cluster (emulated) execution
execute_exchange = run_exchange


def run_baseline(assignment, topo, placement, token_bytes, *, payload_seed: int = 0, mode: str = "analytic",
                 cost=None, expert_fn=identity_expert, materialize: bool = True, dtype: str = "f32",
                 acc: str = "f64", device=None) -> ExchangeResult:
    """The disaggregated pack / all-to-all / unpack shuffle without dedup
    (reference run_baseline, engine.py:552-625): same output bytes as
    ``run_exchange``, every (token, k) row crosses, four rearrangement passes."""
    return run_exchange(assignment, topo, placement, token_bytes, payload_seed=payload_seed, mode=mode, cost=cost,
                        ablate=("dcomm", "planner"), expert_fn=expert_fn, materialize=materialize, dtype=dtype,
                        acc=acc, device=device)
