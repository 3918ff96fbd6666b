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
