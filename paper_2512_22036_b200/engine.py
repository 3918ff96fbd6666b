"""GPU execution of the shuffle: one ``Rank`` per libfusco handle.

Two ways to own ranks:

* ``EmulatedCluster`` — all P ranks in one process on one GPU.  Each rank's
  symmetric region is a separate device allocation and every handle gets the
  table of all P regions, so the *same* kernels that push/pull over NVLink
  here address "peer" memory on the same device.  Phases run rank by rank
  (LOCAL for all, then REMOTE for all), so no kernel ever waits on one that
  has not been launched.  This is the device analogue of the reference's
  one-thread-per-simulated-GPU model (reference engine.py:770-796) and is
  what the drop-in ``run_exchange`` and the parity tests use.
* ``EPBuffer`` — one process per GPU (torchrun), regions exported with CUDA
  IPC and exchanged over ``torch.distributed``; kernels run with
  ``FS_PHASE_ALL`` and synchronise with peers through NVLink flags.

Neither path has a CPU fallback: without libfusco.so every call raises.
"""

from __future__ import annotations

import ctypes
from ctypes import byref, c_int, c_size_t, c_void_p
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import (
    FS_ACC_F32,
    FS_ACC_F64,
    FS_DTYPE_BF16,
    FS_DTYPE_F32,
    FS_NSTATS,
    FS_PHASE_ALL,
    FS_PHASE_LOCAL,
    FS_PHASE_REMOTE,
    FS_SRC_ACT,
    FS_SRC_ACT_OUT,
    call,
    ptr,
    stream_ptr,
)

_DTYPES = {"f32": (torch.float32, FS_DTYPE_F32), "bf16": (torch.bfloat16, FS_DTYPE_BF16)}
_ACCS = {"f32": FS_ACC_F32, "f64": FS_ACC_F64}


def dtype_code(dtype) -> tuple[torch.dtype, int]:
    if isinstance(dtype, str):
        if dtype not in _DTYPES:
            raise ValueError(f"dtype must be one of {sorted(_DTYPES)}")
        return _DTYPES[dtype]
    for tdt, code in _DTYPES.values():
        if dtype == tdt:
            return tdt, code
    raise ValueError(f"unsupported payload dtype {dtype}")


class _DeviceView:
    """Exposes a raw device pointer through __cuda_array_interface__."""

    def __init__(self, address: int, nbytes: int):
        self.__cuda_array_interface__ = {
            "shape": (nbytes,),
            "typestr": "|u1",
            "data": (address, False),
            "version": 3,
            "strides": None,
        }


def wrap_device(address: int, nbytes: int, device: torch.device) -> torch.Tensor:
    """Zero-copy uint8 tensor over device memory the library owns."""
    if nbytes == 0:
        return torch.empty(0, dtype=torch.uint8, device=device)
    with torch.cuda.device(device):
        return torch.as_tensor(_DeviceView(address, nbytes), device=device)


@dataclass
class Plan:
    """Device-resident output of the layout planner for one rank.

    ``row_of[i, k]`` — row of local token i's k-th expert in its owner's
    activation buffer (reference ``_activation_layouts`` row_of,
    planner.py:138-159); ``expert_counts`` / ``expert_offsets`` — this
    rank's per-local-expert run lengths and starts; ``first_mask`` — the
    token-node first-appearance mask (routing.py:86-98); ``rank_mask`` —
    destination-rank bitmask per token; ``stats`` — FS_STAT_* counters.
    """

    rank: int
    epoch: int
    num_tokens: int
    topk_idx: torch.Tensor
    row_of: torch.Tensor
    expert_counts: torch.Tensor
    expert_offsets: torch.Tensor
    first_mask: torch.Tensor | None
    rank_mask: torch.Tensor | None
    stats: torch.Tensor

    @property
    def num_rows(self) -> int:
        return int(self.expert_offsets[-1].item())


class Rank:
    """One expert-parallel rank = one libfusco handle."""

    def __init__(
        self,
        *,
        device: torch.device,
        rank: int,
        world: int,
        num_experts: int,
        topk: int,
        token_bytes: int,
        max_tokens: int,
        owner: np.ndarray,
        node_of: np.ndarray | None,
        regions: list[int],
        max_rows: int,
        with_act_out: bool,
        grid_ctas: int = 0,
        timeout_ms: int = 0,
        nodedup: bool = False,
        balance: bool = True,
    ):
        self.device = torch.device(device)
        self.dev_index = self.device.index if self.device.index is not None else torch.cuda.current_device()
        self.rank, self.world = rank, world
        self.num_experts, self.topk, self.token_bytes = num_experts, topk, token_bytes
        self.max_tokens = max_tokens
        self.owner = np.ascontiguousarray(owner, dtype=np.int32)
        self.local_experts = np.flatnonzero(self.owner == rank).astype(np.int64)
        nodes = None if node_of is None else np.ascontiguousarray(node_of, dtype=np.int32)
        self._node_of = nodes
        peers = (c_void_p * world)(*regions)
        h = c_void_p()
        call(
            "fs_create", self.dev_index, rank, world, num_experts, topk, token_bytes, max_tokens,
            int(max_rows), int(with_act_out),
            self.owner.ctypes.data_as(c_void_p),
            None if nodes is None else nodes.ctypes.data_as(c_void_p),
            peers, int(grid_ctas), int(timeout_ms), byref(h),
        )
        self.handle = h
        if nodedup:  # the reference's planner ablation: every (token, k) row crosses the link
            call("fs_set_nodedup", h, 1)
        if not balance:  # the reference's balancer ablation: static work striding, no rotation
            call("fs_set_balance", h, 0)
        self.with_act_out = bool(with_act_out)
        self.max_rows = int(_lib.load().fs_max_rows(h))
        self.region = regions[rank]
        n = c_int()
        call("fs_grid_ctas", h, byref(n))
        self.grid_ctas = n.value

    # -- lifecycle ----------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "handle", None) is not None and self.handle.value:
            _lib.load().fs_destroy(self.handle)
            self.handle = c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def epoch(self) -> int:
        return int(_lib.load().fs_epoch(self.handle))

    # -- buffers ------------------------------------------------------------
    def buffer(self, which: int) -> torch.Tensor:
        p = c_void_p()
        call("fs_buffer_ptr", self.handle, which, byref(p))
        return wrap_device(p.value, self.max_rows * self.token_bytes, self.device)

    def _rows_view(self, which: int, rows: int | None, dtype: torch.dtype) -> torch.Tensor:
        rows = self.max_rows if rows is None else rows
        if not 0 <= rows <= self.max_rows:
            raise ValueError(f"rows must be in [0, {self.max_rows}]")
        width = self.token_bytes // torch.empty(0, dtype=dtype).element_size()
        return self.buffer(which)[: rows * self.token_bytes].view(dtype).view(rows, width)

    def act(self, rows: int | None = None, dtype: torch.dtype = torch.uint8) -> torch.Tensor:
        """This rank's activation rows of the current epoch, [rows, width]."""
        return self._rows_view(0, rows, dtype)

    def act_out(self, rows: int | None = None, dtype: torch.dtype = torch.uint8) -> torch.Tensor:
        """The symmetric expert-output rows (same row layout as act)."""
        return self._rows_view(1, rows, dtype)

    def _stream(self, stream):
        """The given stream, else the current stream of this rank's device."""
        return stream_ptr(stream if stream is not None else torch.cuda.current_stream(self.device))

    # -- hot path -----------------------------------------------------------
    def new_plan(self, topk_idx: torch.Tensor, with_masks: bool = True) -> Plan:
        T = topk_idx.shape[0]
        dev = self.device
        nloc = self.local_experts.size
        return Plan(
            rank=self.rank,
            epoch=-1,
            num_tokens=T,
            topk_idx=topk_idx,
            row_of=torch.empty((T, self.topk), dtype=torch.int32, device=dev),
            expert_counts=torch.empty(nloc, dtype=torch.int32, device=dev),
            expert_offsets=torch.empty(nloc + 1, dtype=torch.int32, device=dev),
            first_mask=torch.empty((T, self.topk), dtype=torch.uint8, device=dev) if with_masks else None,
            rank_mask=torch.empty(T, dtype=torch.int32, device=dev) if with_masks else None,
            stats=torch.empty(FS_NSTATS, dtype=torch.int64, device=dev),
        )

    def _check_idx(self, topk_idx: torch.Tensor) -> int:
        if topk_idx.dim() != 2 or topk_idx.shape[1] != self.topk:
            raise ValueError(f"topk_idx must be [T, {self.topk}]")
        if topk_idx.dtype not in (torch.int32, torch.int64):
            raise ValueError("topk_idx must be int32 or int64")
        if not topk_idx.is_contiguous() or topk_idx.device != self.device:
            raise ValueError("topk_idx must be contiguous on the rank's device")
        if topk_idx.shape[0] > self.max_tokens:
            raise ValueError(f"{topk_idx.shape[0]} tokens exceed max_tokens={self.max_tokens}")
        return topk_idx.element_size()

    def layout(self, plan: Plan, phase: int = FS_PHASE_ALL, stream=None) -> Plan:
        ib = self._check_idx(plan.topk_idx)
        call(
            "fs_layout", self.handle, ptr(plan.topk_idx), ib, plan.num_tokens, ptr(plan.row_of),
            ptr(plan.expert_counts), ptr(plan.expert_offsets), ptr(plan.first_mask),
            ptr(plan.rank_mask), ptr(plan.stats), phase, self._stream(stream),
        )
        plan.epoch = self.epoch
        return plan

    def dispatch(self, x: torch.Tensor, plan: Plan, phase: int = FS_PHASE_ALL, stream=None,
                 topk_w: torch.Tensor | None = None) -> None:
        """fs_dispatch, or fs_dispatch_w when the router weights are given (the
        owners may then pre-reduce groups of a token's rows for an fp32-
        accumulate combine of this step; include/fusco.h)."""
        if x.shape[0] != plan.num_tokens or x.numel() * x.element_size() != plan.num_tokens * self.token_bytes:
            raise ValueError("x must be [T, token_bytes] bytes matching the plan")
        if not x.is_contiguous() or x.device != self.device:
            raise ValueError("x must be contiguous on the rank's device")
        if plan.epoch != self.epoch:
            raise ValueError("plan is stale: build a new plan (fs_layout) before dispatch")
        if topk_w is None:
            call(
                "fs_dispatch", self.handle, ptr(x), ptr(plan.topk_idx), plan.topk_idx.element_size(),
                ptr(plan.row_of), plan.num_tokens, phase, self._stream(stream),
            )
            return
        if (topk_w.shape != plan.topk_idx.shape or topk_w.dtype not in (torch.float32, torch.float64)
                or not topk_w.is_contiguous() or topk_w.device != self.device):
            raise ValueError("topk_w must be a contiguous f32/f64 [T, K] tensor on the rank's device")
        call(
            "fs_dispatch_w", self.handle, ptr(x), ptr(plan.topk_idx), plan.topk_idx.element_size(),
            ptr(plan.row_of), ptr(topk_w), topk_w.element_size(), plan.num_tokens, phase, self._stream(stream),
        )

    def combine(
        self,
        plan: Plan,
        topk_w: torch.Tensor,
        out: torch.Tensor,
        *,
        dtype_code: int,
        src: int = FS_SRC_ACT,
        acc: int = FS_ACC_F32,
        phase: int = FS_PHASE_ALL,
        stream=None,
    ) -> None:
        if topk_w.shape != (plan.num_tokens, self.topk) or topk_w.dtype not in (torch.float32, torch.float64):
            raise ValueError(f"topk_w must be f32/f64 [T, {self.topk}]")
        if not topk_w.is_contiguous() or not out.is_contiguous():
            raise ValueError("topk_w and out must be contiguous")
        if topk_w.device != self.device or out.device != self.device:
            raise ValueError("topk_w and out must be on the rank's device")
        want_dt = {FS_DTYPE_F32: torch.float32, FS_DTYPE_BF16: torch.bfloat16}.get(dtype_code)
        if want_dt is None or out.dtype != want_dt:
            raise ValueError(f"out must be {want_dt} for dtype_code {dtype_code}")
        if out.numel() * out.element_size() != plan.num_tokens * self.token_bytes:
            raise ValueError("out must hold num_tokens x token_bytes bytes")
        if plan.epoch != self.epoch:
            raise ValueError("plan is stale: combine must follow its own dispatch")
        call(
            "fs_combine", self.handle, ptr(plan.topk_idx), plan.topk_idx.element_size(), ptr(plan.row_of),
            ptr(topk_w), topk_w.element_size(), plan.num_tokens, ptr(out), dtype_code, src, acc, phase,
            self._stream(stream),
        )

    def check(self, stream=None) -> None:
        """Synchronise and raise if a kernel recorded an error (timeout, range)."""
        call("fs_check", self.handle, self._stream(stream))


def region_bytes(world: int, num_experts: int, topk: int, token_bytes: int, max_tokens: int, max_rows: int,
                 with_act_out: bool) -> int:
    n = c_size_t()
    call("fs_region_bytes", world, num_experts, topk, token_bytes, max_tokens, int(max_rows), int(with_act_out),
         byref(n))
    return n.value


def default_max_rows(world: int, max_tokens: int, topk: int, owner: np.ndarray) -> int:
    """Worst case rows one rank can receive: every token of every rank routes
    min(K, experts on that rank) rows to it.  Sized so no host sync is ever
    needed to size buffers (180 GB HBM per GPU makes this affordable)."""
    per_rank = np.bincount(np.asarray(owner, dtype=np.int64), minlength=world)
    return max(1, world * max_tokens * min(topk, int(per_rank.max(initial=1))))


class EmulatedCluster:
    """P ranks on the current GPU (see module docstring).

    ``devices=[d0, d1, ...]`` instead places rank r's region and kernels on
    GPU d_r (one process, peer access enabled between them): the same phased
    launches then move real bytes over NVLink with no kernel waiting on
    another rank's, so a single-process profiler can count each kernel's
    NVLink traffic (tools/ncu_nvlink.py)."""

    def __init__(
        self,
        world: int,
        num_experts: int,
        topk: int,
        token_bytes: int,
        max_tokens: int,
        owner: np.ndarray | None = None,
        node_of: np.ndarray | None = None,
        max_rows: int = 0,
        with_act_out: bool = False,
        grid_ctas: int = 0,
        device: torch.device | str | None = None,
        timeout_ms: int = 0,
        nodedup: bool = False,
        balance: bool = True,
        devices=None,
    ):
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        if devices is not None:
            if len(devices) != world:
                raise ValueError("devices must list one GPU per rank")
            self.devices = [torch.device("cuda", torch.device(d).index if not isinstance(d, int) else d)
                            for d in devices]
            self.device = self.devices[0]
        else:
            self.devices = [self.device] * world
        self.multi_device = len({d.index for d in self.devices}) > 1
        owner = np.arange(num_experts) % world if owner is None else np.asarray(owner)
        self.world = world
        self.token_bytes = token_bytes
        self.topk = topk
        self.owner = owner
        mr = max_rows or default_max_rows(world, max_tokens, topk, owner)
        nbytes = region_bytes(world, num_experts, topk, token_bytes, max_tokens, mr, with_act_out)
        self.regions: list[int] = []
        for r in range(world):
            p = c_void_p()
            call("fs_sym_alloc", self.devices[r].index, nbytes, byref(p))
            self.regions.append(p.value)
        if self.multi_device:
            idx = sorted({d.index for d in self.devices})
            for a in idx:
                for b in idx:
                    if a != b:
                        call("fs_enable_peer_access", a, b)
        self.ranks = [
            Rank(
                device=self.devices[r], rank=r, world=world, num_experts=num_experts, topk=topk,
                token_bytes=token_bytes, max_tokens=max_tokens, owner=owner, node_of=node_of,
                regions=self.regions, max_rows=mr, with_act_out=with_act_out, grid_ctas=grid_ctas,
                timeout_ms=timeout_ms, nodedup=nodedup, balance=balance,
            )
            for r in range(world)
        ]

    def close(self) -> None:
        for r in getattr(self, "ranks", []):
            r.close()
        for d, p in zip(getattr(self, "devices", []), getattr(self, "regions", [])):
            _lib.load().fs_sym_free(d.index, c_void_p(p))
        self.ranks, self.regions = [], []

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # A single rank has no peer to wait for: it runs the production launches
    # (FS_PHASE_ALL, e.g. the one-cluster planner).  P > 1 runs every rank's
    # LOCAL phase, then every rank's REMOTE phase.
    def _phases(self):
        return (FS_PHASE_ALL,) if self.world == 1 else (FS_PHASE_LOCAL, FS_PHASE_REMOTE)

    def layout(self, topk_idx: list[torch.Tensor], with_masks: bool = True) -> list[Plan]:
        return self.layout_into([r.new_plan(t, with_masks) for r, t in zip(self.ranks, topk_idx)])

    def _phase_done(self) -> None:
        """Across GPUs, a phase of every rank completes before the next starts
        (on one GPU the stream order already guarantees it)."""
        if self.multi_device:
            for d in sorted({d.index for d in self.devices}):
                torch.cuda.synchronize(d)

    def layout_into(self, plans: list[Plan]) -> list[Plan]:
        """Re-plan into existing Plan tensors (same routing tensors; e.g. a graph-captured step)."""
        for ph in self._phases():
            for r, p in zip(self.ranks, plans):
                r.layout(p, ph)
            self._phase_done()
        return plans

    def dispatch(self, xs: list[torch.Tensor], plans: list[Plan], ws: list[torch.Tensor] | None = None) -> None:
        for ph in self._phases():
            for j, (r, x, p) in enumerate(zip(self.ranks, xs, plans)):
                r.dispatch(x, p, ph, topk_w=None if ws is None else ws[j])
            self._phase_done()

    def combine(self, plans, ws, outs, *, dtype_code: int, src: int = FS_SRC_ACT, acc: int = FS_ACC_F32):
        for ph in self._phases():
            for r, p, w, o in zip(self.ranks, plans, ws, outs):
                r.combine(p, w, o, dtype_code=dtype_code, src=src, acc=acc, phase=ph)
            self._phase_done()

    def check(self) -> None:
        for r in self.ranks:
            r.check()


@dataclass
class _Peers:
    regions: list[int] = field(default_factory=list)
    opened: list[int] = field(default_factory=list)


class EPBuffer:
    """Per-process expert-parallel shuffle over NVLink (one rank per GPU).

    SPEC.md's ``build_plan`` / ``execute_dispatch`` / ``execute_combine``
     for one rank of a real multi-GPU job::

        buf = EPBuffer(group, num_experts=256, topk=8, hidden=7168, dtype="bf16",
                       max_tokens=4096)
        plan = buf.build_plan(topk_idx)            # on-device layout planner
        act = buf.dispatch(x, plan)                # [rows, hidden], expert-major
        y = buf.expert_out(plan.num_rows)          # write expert outputs here ...
        out = buf.combine(plan, topk_w)            # ... or pass src="act"
    """

    def __init__(
        self,
        group=None,
        *,
        num_experts: int,
        topk: int,
        hidden: int,
        dtype="bf16",
        max_tokens: int,
        owner: np.ndarray | None = None,
        max_rows: int = 0,
        with_act_out: bool = True,
        grid_ctas: int = 0,
        timeout_ms: int = 0,
        exchange=None,
        balance: bool = True,
    ):
        import torch.distributed as dist

        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.world = dist.get_world_size(group)
            self.rank_id = dist.get_rank(group)
        else:  # single-GPU job: one rank, nothing to exchange
            self.world, self.rank_id = 1, 0
            exchange = exchange or (lambda obj, grp: [obj])
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.dtype, self.dtype_code = dtype_code(dtype)
        self.hidden = hidden
        elem = torch.empty(0, dtype=self.dtype).element_size()
        token_bytes = hidden * elem
        owner = np.arange(num_experts) % self.world if owner is None else np.asarray(owner)
        mr = max_rows or default_max_rows(self.world, max_tokens, topk, owner)
        nbytes = region_bytes(self.world, num_experts, topk, token_bytes, max_tokens, mr, with_act_out)
        cfg = (self.world, num_experts, topk, token_bytes, max_tokens, int(mr), bool(with_act_out),
               tuple(int(o) for o in owner), int(grid_ctas))
        own = c_void_p()
        call("fs_sym_alloc", self.device.index, nbytes, byref(own))
        self._peers = _Peers()
        try:
            handle = (ctypes.c_uint8 * 64)()
            call("fs_ipc_handle", self.device.index, own, handle)
            infos = bootstrap_exchange(bytes(handle), cfg, self.rank_id, group, exchange)
            for g, h in enumerate(infos):
                if g == self.rank_id:
                    self._peers.regions.append(own.value)
                    continue
                p = c_void_p()
                raw = (ctypes.c_uint8 * 64).from_buffer_copy(h)
                call("fs_ipc_open", self.device.index, raw, byref(p))
                self._peers.regions.append(p.value)
                self._peers.opened.append(p.value)
            self.r = Rank(
                device=self.device, rank=self.rank_id, world=self.world, num_experts=num_experts, topk=topk,
                token_bytes=token_bytes, max_tokens=max_tokens, owner=owner, node_of=None,
                regions=self._peers.regions, max_rows=mr, with_act_out=with_act_out, grid_ctas=grid_ctas,
                timeout_ms=timeout_ms, balance=balance,
            )
        except BaseException:  # release what was mapped / allocated before re-raising
            lib = _lib.load()
            for p in self._peers.opened:
                lib.fs_ipc_close(self.device.index, c_void_p(p))
            lib.fs_sym_free(self.device.index, own)
            raise
        self._own = own.value
        self.with_act_out = with_act_out
        self._closed = False

    # SPEC names
    def build_plan(self, topk_idx: torch.Tensor, with_masks: bool = False, stream=None) -> Plan:
        plan = self.r.new_plan(topk_idx, with_masks)
        return self.r.layout(plan, FS_PHASE_ALL, stream)

    def dispatch(self, x: torch.Tensor, plan: Plan, stream=None, rows: int | None = None,
                 topk_w: torch.Tensor | None = None) -> torch.Tensor:
        """Returns this rank's activation view [rows, hidden] (rows = max_rows
        unless given; the valid prefix is plan.expert_offsets[-1]).  With the
        router weights (the ones the combine will get), an fp32-accumulate
        combine of this step lets each owner pre-reduce groups of >= 3 of a
        token's rows (>= 2 for fp32 rows) into one fp32 partial."""
        if x.dtype != self.dtype or x.dim() != 2 or x.shape[1] != self.hidden:
            raise ValueError(f"x must be [T, {self.hidden}] {self.dtype}")
        self.r.dispatch(x, plan, FS_PHASE_ALL, stream, topk_w=topk_w)
        return self.r.act(rows, self.dtype)

    execute_dispatch = dispatch

    def expert_out(self, rows: int | None = None) -> torch.Tensor:
        return self.r.act_out(rows, self.dtype)

    def combine(self, plan: Plan, topk_w: torch.Tensor, out: torch.Tensor | None = None, *, src: str = "act_out",
                acc: str = "f32", stream=None) -> torch.Tensor:
        if out is None:
            out = torch.empty((plan.num_tokens, self.hidden), dtype=self.dtype, device=self.device)
        code = FS_SRC_ACT_OUT if src == "act_out" else FS_SRC_ACT
        self.r.combine(plan, topk_w, out, dtype_code=self.dtype_code, src=code, acc=_ACCS[acc], phase=FS_PHASE_ALL,
                       stream=stream)
        return out

    execute_combine = combine

    def check(self, stream=None) -> None:
        self.r.check(stream)

    def close(self) -> None:
        if getattr(self, "_closed", True):
            return
        self._closed = True
        self.r.close()
        lib = _lib.load()
        for p in self._peers.opened:
            lib.fs_ipc_close(self.device.index, c_void_p(p))
        lib.fs_sym_free(self.device.index, c_void_p(self._own))

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def bootstrap_exchange(handle: bytes, cfg: tuple, rank: int, group=None, exchange=None) -> list[bytes]:
    """All-gather every rank's 64-byte region handle together with its shuffle
    configuration; every rank must agree on the configuration (the symmetric
    regions have identical layouts), else ValueError on every rank.  Returns the
    handles in rank order."""
    gather = exchange or exchange_objects
    infos = gather((bytes(handle), cfg, rank), group)
    for i, (h, c, r) in enumerate(infos):
        if r != i:
            raise ValueError(f"bootstrap: slot {i} answered by rank {r}")
        if c != cfg:
            raise ValueError(f"rank {r} shuffle configuration differs from rank {rank}")
        if len(h) != 64:
            raise ValueError(f"rank {r} sent a malformed region handle")
    return [h for h, _, _ in infos]


def exchange_objects(obj, group=None) -> list:
    """All-gather a picklable object over torch.distributed (bootstrap only)."""
    import torch.distributed as dist

    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, obj, group=group)
    return out
