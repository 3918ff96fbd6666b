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
    dtype: str = "f32"           # payload element type of the rows ("f32" as in the reference, or "bf16")
    # the resident device state the executors run on (shared by the dispatch
    # and combine plans of one routing); None for a host-only plan
    execution: object = field(default=None, repr=False, compare=False)


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

    def __init__(self, assignment, topo, placement, token_bytes, *, with_act_out, device=None, nodedup=False,
                 dtype="f32", balance=True):
        self.dtype = dtype
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
            nodedup=nodedup, balance=balance,
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
            loads=loads, dtype=self.dtype,
        )


def _open_session(assignment, topo, placement, token_bytes, ablate, *, with_act_out, device=None) -> _Session:
    """A session whose ranks push without dedup when ``planner`` is ablated
    (every (token, k) row crosses the link, ``fs_set_nodedup``) and stride
    their work statically when ``balancer`` is ablated (``fs_set_balance``)."""
    return _Session(assignment, topo, placement, token_bytes, with_act_out=with_act_out, device=device,
                    nodedup="planner" in ablate, balance="balancer" not in ablate)


def build_plan_pair(
    assignment: RoutingAssignment,
    topo: ClusterTopology,
    placement: ExpertPlacement,
    token_bytes: int,
    balancer: str = "greedy",
    device=None,
    dtype: str = "f32",
) -> tuple[GpuPlan, GpuPlan, np.ndarray]:
    """Device-planned (dispatch, combine, groups) (reference planner.py:485-497):
    loads, then groups, then both directions.  The plans stay executable
    (``allocate_buffers`` / ``apply_*`` / ``execute_*`` below) for as long as
    they are alive."""
    _validate(assignment, topo, placement, token_bytes)
    ex = _execution(assignment, topo, placement, token_bytes, nodedup=False, device=device, dtype=dtype)
    d = ex.host_plan("dispatch", None)
    groups = _balancer.build_groups(balancer, d.loads, topo)
    d.groups = groups
    c = ex.host_plan("combine", groups)
    return d, c, groups


def build_dispatch_plan(assignment, topo, placement, token_bytes, groups, device=None, dtype: str = "f32") -> GpuPlan:
    """Deduplicated dispatch plan for a fixed group assignment (reference
    planner.py:211-339): the device layout planner's row order, per-rank
    dedup counters and first mask; executable by ``apply_node_level`` /
    ``apply_expert_level`` / ``execute_dispatch``."""
    _validate(assignment, topo, placement, token_bytes)
    _balancer.validate_groups(groups, topo)
    ex = _execution(assignment, topo, placement, token_bytes, nodedup=False, device=device, dtype=dtype)
    return ex.host_plan("dispatch", np.asarray(groups))


def build_combine_plan(assignment, topo, placement, token_bytes, groups, device=None, dtype: str = "f32") -> GpuPlan:
    """Return-path plan, no dedup (reference planner.py:342-482): the same
    device layout, read back by the pull combine; ``reduce_weights`` per
    source rank.  Executable by ``reduce_outputs`` / ``execute_combine``."""
    _validate(assignment, topo, placement, token_bytes)
    _balancer.validate_groups(groups, topo)
    ex = _execution(assignment, topo, placement, token_bytes, nodedup=False, device=device, dtype=dtype)
    return ex.host_plan("combine", np.asarray(groups))


def build_direct_plans(assignment, topo, placement, token_bytes, device=None, dtype: str = "f32"):
    """The planner ablation's plans (reference planner.py:563-659): same
    layouts, no dedup — every remote (token, expert) row crosses the link
    (the device push with ``fs_set_nodedup``)."""
    _validate(assignment, topo, placement, token_bytes)
    ex = _execution(assignment, topo, placement, token_bytes, nodedup=True, device=device, dtype=dtype)
    d = ex.host_plan("dispatch", None)
    d.inter_bytes_total = naive_inter_node_bytes(assignment, placement, topo, token_bytes)
    return d, ex.host_plan("combine", None)


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
    execute the real kernels and report CUDA-event times.  Ablations:
    ``planner`` pushes every (token, k) row (no dedup), ``balancer`` turns
    the device balancing off (static work striding, no rotation) and the
    groups to "static", ``dcomm`` runs the disaggregated pack / all-to-all /
    unpack baseline.
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


# ---------------------------------------------------------------------------
# The reference's executor API (engine.py:249-338) over the
# resident device state of a plan pair.
#
# Buffers are a dict ``"kind/rank" -> flat uint8 device tensor`` as in the
# reference (``planner.py:35-49``).  ``allocate_buffers`` returns
# ``token/s`` and ``output/s`` (plain device tensors) and ``activation/g`` /
# ``act_out/g`` — views of rank g's symmetric region, because the dispatch
# writes every owner's expert-major rows in place over NVLink.  The
# reference's landing and staging kinds (``fwd_recv``, ``comb_recv``,
# ``staging``) do not exist here: no byte is staged between the token rows
# and the expert-major rows, nor between the expert outputs and the
# reduction.  Stage mapping (each a launch of the fused kernels' phase):
#
#   dispatch  apply_node_level    push of every (token, destination rank) row
#                                 to its owner (one crossing per rank)
#             apply_expert_level  receiver fan-out of a token's further rows
#                                 on the same rank
#   combine   apply_expert_level  owners publish "expert outputs ready"
#             apply_node_level    (nothing left to move: the pull is fused
#                                 into the reduction)
#             reduce_outputs      pull of the K rows + k-ascending weighted sum
# ---------------------------------------------------------------------------

import hashlib as _hashlib
import weakref as _weakref

from ._lib import FS_PHASE_LOCAL, FS_PHASE_REMOTE, FS_ACC_F64

_EXECUTIONS: "_weakref.WeakValueDictionary" = _weakref.WeakValueDictionary()


def _fingerprint(assignment, placement) -> str:
    h = _hashlib.sha1()
    for arr in (assignment.experts, assignment.source, placement.owner):
        h.update(np.ascontiguousarray(arr, dtype=np.int64).tobytes())
        h.update(b"|")
    return h.hexdigest()


class _Execution:
    """A planned shuffle resident on the device: the emulated cluster, its
    per-rank device plans, and which stages of the current epoch have run."""

    def __init__(self, assignment, topo, placement, token_bytes, *, nodedup, device, dtype):
        self.sess = _Session(assignment, topo, placement, token_bytes, with_act_out=True, device=device,
                             nodedup=nodedup, dtype=dtype)
        self.plans = self.sess.plans()
        self.sess.cluster.check()
        self.tdt, self.code = dtype_code(dtype)
        self.stage: set[str] = set()

    def host_plan(self, direction, groups) -> GpuPlan:
        p = self.sess.host_plan(self.plans, direction, groups)
        p.execution = self
        return p

    def replan(self) -> None:
        """A new epoch of the same routing (the device plan is recomputed)."""
        self.sess.cluster.layout_into(self.plans)
        self.sess.cluster.check()
        self.stage.clear()

    @property
    def ranks(self):
        return self.sess.cluster.ranks

    def rows(self, g: int) -> int:
        return self.plans[g].num_rows

    def close(self) -> None:
        self.sess.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _execution(assignment, topo, placement, token_bytes, *, nodedup, device, dtype) -> _Execution:
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    key = (_fingerprint(assignment, placement), topo.num_nodes, topo.gpus_per_node, int(token_bytes),
           bool(nodedup), str(dev), dtype)
    ex = _EXECUTIONS.get(key)
    if ex is None:
        ex = _Execution(assignment, topo, placement, token_bytes, nodedup=nodedup, device=dev, dtype=dtype)
        _EXECUTIONS[key] = ex
    return ex


def _exec_of(plan) -> _Execution:
    ex = getattr(plan, "execution", None)
    if ex is None:
        raise ValueError("plan has no device state: build it with build_plan_pair / build_dispatch_plan / "
                         "build_combine_plan")
    return ex


def allocate_buffers(*plans: GpuPlan) -> dict[str, torch.Tensor]:
    """Buffers for a plan pair (reference engine.py:249-254), sized by the
    plans: ``token/s``, ``output/s`` zero-filled device tensors,
    ``activation/g`` / ``act_out/g`` views of rank g's symmetric rows."""
    if not plans:
        raise ValueError("allocate_buffers needs at least one plan")
    ex = _exec_of(plans[0])
    if any(_exec_of(p) is not ex for p in plans):
        raise ValueError("plans of different routings cannot share buffers")
    tb, dev = plans[0].token_bytes, ex.sess.dev
    bufs: dict[str, torch.Tensor] = {}
    for s, ids in enumerate(ex.sess.ids):
        bufs[f"token/{s}"] = torch.zeros(ids.size * tb, dtype=torch.uint8, device=dev)
        bufs[f"output/{s}"] = torch.zeros(ids.size * tb, dtype=torch.uint8, device=dev)
    for g, r in enumerate(ex.ranks):
        n = ex.rows(g)
        bufs[f"activation/{g}"] = r.act(n).reshape(-1)
        bufs[f"act_out/{g}"] = r.act_out(n).reshape(-1)
    return bufs


def _buf(buffers, kind: str, g: int, nbytes: int, region: torch.Tensor | None = None) -> torch.Tensor:
    name = f"{kind}/{g}"
    if name not in buffers:
        raise ValueError(f"missing buffer {name}")
    b = buffers[name]
    if not isinstance(b, torch.Tensor) or not b.is_cuda or b.dtype != torch.uint8 or not b.is_contiguous():
        raise ValueError(f"buffer {name} must be a contiguous uint8 CUDA tensor (allocate_buffers)")
    if b.numel() != nbytes:
        raise ValueError(f"buffer {name} holds {b.numel()} bytes, the plan needs {nbytes}")
    if region is not None and b.data_ptr() != region.data_ptr():
        raise ValueError(f"buffer {name} must be the symmetric-region view from allocate_buffers "
                         "(peers write these rows in place)")
    return b


def fill_token_buffers(plan: GpuPlan, buffers, payloads) -> None:
    """token/s = payload rows of source s's tokens, ascending global id
    (reference engine.py:257-263)."""
    ex, tb = _exec_of(plan), plan.token_bytes
    pay = torch.as_tensor(np.ascontiguousarray(payloads).reshape(plan.num_tokens, tb)) \
        if not isinstance(payloads, torch.Tensor) else payloads.reshape(plan.num_tokens, tb)
    for s, ids in enumerate(ex.sess.ids):
        if ids.size:
            dst = _buf(buffers, "token", s, ids.size * tb).view(ids.size, tb)
            dst.copy_(pay[torch.as_tensor(ids, device=pay.device)])


def _tokens(ex, buffers, tb):
    return [_buf(buffers, "token", s, ids.size * tb).view(ids.size, tb) for s, ids in enumerate(ex.sess.ids)]


def _check_region_bufs(ex, buffers, kind, tb):
    for g, r in enumerate(ex.ranks):
        n = ex.rows(g)
        _buf(buffers, kind, g, n * tb, r.act(n) if kind == "activation" else r.act_out(n))


def apply_node_level(plan: GpuPlan, buffers) -> None:
    """Dispatch: push every (token, destination rank) row into its owner's
    expert-major rows (reference engine.py:266-269).  Combine: no separate
    movement (the pull is fused into ``reduce_outputs``)."""
    ex, tb = _exec_of(plan), plan.token_bytes
    if plan.direction == "dispatch":
        xs = _tokens(ex, buffers, tb)
        _check_region_bufs(ex, buffers, "activation", tb)
        if "d_node" in ex.stage:  # a repeated dispatch of the same routing: a new epoch
            ex.replan()
        for r, x, p in zip(ex.ranks, xs, ex.plans):
            r.dispatch(x, p, FS_PHASE_LOCAL)
        ex.stage.add("d_node")
        return
    if "c_expert" not in ex.stage:
        raise ValueError("combine: apply_expert_level first (expert outputs leave their owners first)")
    ex.stage.add("c_node")


def apply_expert_level(plan: GpuPlan, buffers) -> None:
    """Dispatch: receiver fan-out of each token's further rows on the same
    rank (reference engine.py:272-276).  Combine: owners publish their
    expert outputs to the pulling ranks."""
    ex, tb = _exec_of(plan), plan.token_bytes
    if plan.direction == "dispatch":
        if "d_node" not in ex.stage or "d_expert" in ex.stage:
            raise ValueError("dispatch: apply_node_level first (once per expert-level pass)")
        xs = _tokens(ex, buffers, tb)
        for r, x, p in zip(ex.ranks, xs, ex.plans):
            r.dispatch(x, p, FS_PHASE_REMOTE)
        ex.sess.cluster.check()
        ex.stage.add("d_expert")
        return
    if "d_expert" not in ex.stage:
        raise ValueError("combine before dispatch")
    _combine_phase(ex, plan, buffers, FS_PHASE_LOCAL, None)
    ex.stage.add("c_expert")


def run_experts(plan: GpuPlan, buffers, expert_fn) -> None:
    """activation -> act_out on every rank through the row-aligned expert map
    (reference engine.py:295-310).  ``expert_fn(act_f32 [rows, width] CUDA
    tensor, expert_ids [rows] CUDA int64) -> [rows, width]``."""
    ex, tb = _exec_of(plan), plan.token_bytes
    if "d_expert" not in ex.stage:
        raise ValueError("run_experts before the dispatch completed")
    _check_region_bufs(ex, buffers, "activation", tb)
    _check_region_bufs(ex, buffers, "act_out", tb)
    dev = ex.sess.dev
    for g, (r, p) in enumerate(zip(ex.ranks, ex.plans)):
        n = ex.rows(g)
        if n == 0:
            continue
        eids = torch.repeat_interleave(torch.as_tensor(r.local_experts, device=dev), p.expert_counts.to(torch.int64))
        act = r.act(n, ex.tdt)
        y = expert_fn(act.to(torch.float32), eids)
        if not isinstance(y, torch.Tensor) or tuple(y.shape) != tuple(act.shape):
            raise ValueError("expert function must return a tensor of the activation shape")
        r.act_out(n, ex.tdt).copy_(y.to(ex.tdt))
    ex.stage.add("experts")


def _weights_for(ex, plan, s, weights):
    if weights is None:
        w = plan.reduce_weights[s]
    elif isinstance(weights, dict):
        w = weights[s]
    else:
        w = np.asarray(weights)[ex.sess.ids[s]]
    return torch.as_tensor(np.ascontiguousarray(w, dtype=np.float64), device=ex.sess.dev)


def _combine_phase(ex, plan, buffers, phase, weights):
    tb = plan.token_bytes
    width = tb // torch.empty(0, dtype=ex.tdt).element_size()
    src = FS_SRC_ACT_OUT if "experts" in ex.stage else FS_SRC_ACT
    for s, (r, p) in enumerate(zip(ex.ranks, ex.plans)):
        n = ex.sess.ids[s].size
        out = _buf(buffers, "output", s, n * tb).view(ex.tdt).view(n, width)
        r.combine(p, _weights_for(ex, plan, s, weights), out, dtype_code=ex.code, src=src, acc=FS_ACC_F64,
                  phase=phase)


def reduce_outputs(plan: GpuPlan, buffers, weights=None) -> None:
    """output/s[t] = Σ_k w[t,k]·(expert output of (t,k)), f64, k ascending,
    one rounding (reference engine.py:313-338), pulled straight from the
    owners' rows.  ``weights`` overrides ``plan.reduce_weights`` ([T, K]
    global or a per-source dict)."""
    if plan.reduce_weights is None:
        raise ValueError("not a combine plan")
    ex = _exec_of(plan)
    if "d_expert" not in ex.stage:
        raise ValueError("combine before dispatch")
    if "c_expert" not in ex.stage:
        apply_expert_level(plan, buffers)
    _combine_phase(ex, plan, buffers, FS_PHASE_REMOTE, weights)
    ex.sess.cluster.check()
    ex.stage.add("reduced")


def _timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e-3


def execute_dispatch(plan: GpuPlan, buffers, mode: str = "analytic"):
    """run the dispatch plan: returns ({g: activation rows}, PhaseReport)."""
    if plan.direction != "dispatch":
        raise ValueError("not a dispatch plan")
    if mode not in ("analytic", "wallclock"):
        raise ValueError(f"unknown mode {mode!r}")

    def run():
        apply_node_level(plan, buffers)
        apply_expert_level(plan, buffers)

    t = _timed(run)
    acts = {g: buffers[f"activation/{g}"] for g in range(len(_exec_of(plan).ranks))}
    rep = PhaseReport("dispatch", mode, 0.0, 0.0, t, plan.inter_bytes_total, plan.intra_bytes_total,
                      plan.intra_gpu_bytes, 0)
    return acts, rep


def execute_combine(combine_plan: GpuPlan, activation_out_buffers, weights=None, mode: str = "analytic"):
    """run the combine plan over the expert outputs: returns
    ({s: output rows}, PhaseReport).  The reduction uses ``weights`` ([T, K]
    or per-source) when given, else the plan's ``reduce_weights``."""
    if combine_plan.direction != "combine":
        raise ValueError("not a combine plan")

    def run():
        apply_expert_level(combine_plan, activation_out_buffers)
        apply_node_level(combine_plan, activation_out_buffers)
        reduce_outputs(combine_plan, activation_out_buffers, weights)

    t = _timed(run)
    outs = {s: activation_out_buffers[f"output/{s}"] for s in range(len(_exec_of(combine_plan).ranks))}
    rep = PhaseReport("combine", mode, 0.0, 0.0, t, combine_plan.inter_bytes_total, combine_plan.intra_bytes_total,
                      combine_plan.intra_gpu_bytes, 0)
    return outs, rep
