"""Disaggregated GPU baseline: pack -> NCCL all-to-all -> unpack.

The design Fusco's fused engine replaces, built from stock PyTorch/NCCL on
B200 for an in-box comparison (reference ``run_baseline``,
engine.py:552-625, with the direct no-dedup plans of planner.py:563-659 and
the paper's Table 1 pipeline):

  dispatch  1. index_select token rows into destination-rank-major order
               (one row per (token, k): no deduplication)
            2. NCCL all_to_all_single of the row counts (host sync for splits)
            3. NCCL all_to_all_single of rows and (expert, token) metadata
            4. index_select the received rows into expert-major order
  combine   the mirror: index_copy back to received order, all-to-all back,
            index_copy into (token, k) staging, fp32 weighted sum over k.

Four standalone rearrangement passes per round trip (``rearrange_bytes`` =
4·T·K·tb, reference engine.py:628-630) and a host synchronisation; the fused
path has neither.  Activations come out byte-identical to the fused path's
(same expert-major layout); outputs equal within the combine tolerance.
This module is a measured comparison point, not the product path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch


@dataclass
class BaselineState:
    order: torch.Tensor        # [T*K] (token, k) pairs in destination-rank-major order
    send_splits: list[int]
    recv_splits: list[int]
    perm: torch.Tensor         # received row -> expert-major row order
    num_tokens: int


class DisaggregatedShuffle:
    def __init__(self, group=None, *, num_experts: int, topk: int, owner: np.ndarray | None = None,
                 device: torch.device | None = None):
        import torch.distributed as dist

        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        else:
            self.world, self.rank = 1, 0
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        owner = np.arange(num_experts) % self.world if owner is None else np.asarray(owner)
        self.owner = torch.as_tensor(owner, dtype=torch.int64, device=self.device)
        self.E, self.K = num_experts, topk

    def _a2a(self, out, inp, out_splits, in_splits):
        import torch.distributed as dist

        if self.world == 1:
            out.copy_(inp)
        else:
            dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)

    def dispatch(self, x: torch.Tensor, topk_idx: torch.Tensor) -> tuple[torch.Tensor, BaselineState]:
        T, K = topk_idx.shape
        P = self.world
        flat_e = topk_idx.reshape(-1).to(torch.int64)
        dest = self.owner[flat_e]
        order = torch.argsort(dest, stable=True)                       # (t,k) pairs, rank-major
        tok = torch.div(order, K, rounding_mode="floor")
        send_counts = torch.bincount(dest, minlength=P)
        x_packed = x.index_select(0, tok)                              # rearrangement 1 (pack)
        meta = torch.stack([flat_e[order], tok], 1).to(torch.int32).contiguous()
        recv_counts = torch.empty_like(send_counts)
        self._a2a(recv_counts, send_counts, None, None)
        send_splits = send_counts.tolist()                             # host sync
        recv_splits = recv_counts.tolist()
        n_recv = int(sum(recv_splits))
        x_recv = torch.empty((n_recv, x.shape[1]), dtype=x.dtype, device=x.device)
        meta_recv = torch.empty((n_recv, 2), dtype=torch.int32, device=x.device)
        self._a2a(x_recv, x_packed, recv_splits, send_splits)          # the all-to-all
        self._a2a(meta_recv, meta, recv_splits, send_splits)
        src = torch.repeat_interleave(torch.arange(P, device=x.device),
                                      torch.as_tensor(recv_splits, device=x.device))
        e = meta_recv[:, 0].to(torch.int64)
        t = meta_recv[:, 1].to(torch.int64)
        big = int(T) + 1
        tmax = torch.tensor(big, device=x.device)
        if P > 1:  # token-count bound across ranks for the sort key
            import torch.distributed as dist

            dist.all_reduce(tmax, op=dist.ReduceOp.MAX, group=self.group)
        tm = int(tmax.item())
        perm = torch.argsort((e * P + src) * tm + t)                    # (expert, source, token)
        act = x_recv.index_select(0, perm)                             # rearrangement 2 (unpack)
        return act, BaselineState(order, send_splits, recv_splits, perm, T)

    def combine(self, act_out: torch.Tensor, st: BaselineState, topk_w: torch.Tensor) -> torch.Tensor:
        H = act_out.shape[1]
        y_recv = torch.empty_like(act_out)
        y_recv.index_copy_(0, st.perm, act_out)                        # rearrangement 3
        y_send = torch.empty((st.order.numel(), H), dtype=act_out.dtype, device=act_out.device)
        self._a2a(y_send, y_recv, st.send_splits, st.recv_splits)
        staging = torch.empty_like(y_send)
        staging.index_copy_(0, st.order, y_send)                       # rearrangement 4 (unpack)
        stg = staging.view(st.num_tokens, self.K, H).float()
        acc = torch.zeros((st.num_tokens, H), dtype=torch.float32, device=act_out.device)
        for k in range(self.K):  # k ascending, fp32 (same order as the fused kernel)
            acc.addcmul_(stg[:, k], topk_w[:, k : k + 1].float())
        return acc.to(act_out.dtype)

    @staticmethod
    def rearrange_bytes(num_tokens: int, topk: int, token_bytes: int) -> int:
        """Four standalone passes over the routed rows (engine.py:628-630)."""
        return 4 * num_tokens * topk * token_bytes


def emulated_exchange(xs, idxs, ws, owner, P: int, expert_fn=None, dtype=torch.float32, acc: str = "f32",
                      stream_events: bool = True):
    """Disaggregated shuffle of P emulated ranks on one GPU (the reference's
    ``run_baseline`` executed with stock torch ops): per source rank an
    index_select pack into destination-major order, the "all-to-all" as the
    per-destination concatenation of every source's slice, an index_select
    unpack into (expert, source, token) order; combine mirrors it and reduces
    in k order (f64 multiply-then-add with ``acc="f64"``, as engine.py:322-331).

    Returns (activations per rank [rows, H], outputs per rank [T_s, H],
    (pack+unpack seconds, exchange seconds) per direction).
    """
    dev = xs[0].device
    owner_t = torch.as_tensor(np.asarray(owner), dtype=torch.int64, device=dev)
    K = idxs[0].shape[1] if idxs else 1
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(9)]
    ev[0].record()
    # ---- dispatch: pack per source ----
    packs, metas, counts = [], [], []
    for s in range(P):
        flat_e = idxs[s].reshape(-1).to(torch.int64)
        dest = owner_t[flat_e]
        order = torch.argsort(dest, stable=True)
        tok = torch.div(order, K, rounding_mode="floor")
        packs.append(xs[s].index_select(0, tok))
        metas.append((flat_e[order], tok, order))
        counts.append(torch.bincount(dest, minlength=P).tolist())
    ev[1].record()
    # ---- exchange: destination g receives every source's slice, source order ----
    recv, recv_meta = [], []
    for g in range(P):
        parts, e_l, s_l, t_l = [], [], [], []
        for s in range(P):
            lo = sum(counts[s][:g])
            n = counts[s][g]
            parts.append(packs[s][lo:lo + n])
            e_l.append(metas[s][0][lo:lo + n])
            t_l.append(metas[s][1][lo:lo + n])
            s_l.append(torch.full((n,), s, dtype=torch.int64, device=dev))
        recv.append(torch.cat(parts) if parts else packs[0][:0])
        recv_meta.append((torch.cat(e_l), torch.cat(s_l), torch.cat(t_l)))
    ev[2].record()
    # ---- unpack into expert-major order ----
    acts, perms = [], []
    tmax = max([int(x.shape[0]) for x in xs] + [1]) + 1
    for g in range(P):
        e, src, t = recv_meta[g]
        perm = torch.argsort((e * P + src) * tmax + t)
        acts.append(recv[g].index_select(0, perm))
        perms.append(perm)
    ev[3].record()
    outs_act = acts
    if expert_fn is not None:
        outs_act = []
        for g in range(P):
            eids = recv_meta[g][0].index_select(0, perms[g])
            y = expert_fn(acts[g].to(torch.float32), eids)
            outs_act.append(y.to(acts[g].dtype))
    ev[4].record()
    # ---- combine: back to received order, exchange back, unpack to (t, k) ----
    back = []
    for g in range(P):
        y = torch.empty_like(outs_act[g])
        y.index_copy_(0, perms[g], outs_act[g])
        back.append(y)
    ev[5].record()
    staged = []
    for s in range(P):
        parts = []
        for g in range(P):
            lo = sum(counts[q][g] for q in range(s))
            parts.append(back[g][lo:lo + counts[s][g]])
        staged.append(torch.cat(parts) if parts else back[0][:0])
    ev[6].record()
    outs = []
    for s in range(P):
        T = xs[s].shape[0]
        H = xs[s].shape[1]
        stg = torch.empty((T * K, H), dtype=staged[s].dtype, device=dev)
        stg.index_copy_(0, metas[s][2], staged[s])
        stg = stg.view(T, K, H)
        w = ws[s]
        if acc == "f64":
            out = torch.zeros((T, H), dtype=torch.float64, device=dev)
            for k in range(K):
                out = out + w[:, k : k + 1].double() * stg[:, k].double()
        else:
            out = torch.zeros((T, H), dtype=torch.float32, device=dev)
            for k in range(K):
                out.addcmul_(stg[:, k].float(), w[:, k : k + 1].float())
        outs.append(out.to(dtype))
    ev[7].record()
    torch.cuda.synchronize()
    t = lambda i, j: ev[i].elapsed_time(ev[j]) * 1e-3  # noqa: E731
    return acts, outs, ((t(0, 1) + t(2, 3), t(1, 2)), (t(4, 5) + t(6, 7), t(5, 6)))
