"""Wire and golden formats of a plan (§8f next row #4).

* Descriptor tables (reference ``DescriptorList.to_bytes/from_bytes``,
  descriptor.py:224-241): little-endian u64 count, then (offset, length) u64
  pairs.
* ``plan_to_json`` (reference planner.py:676-730, the ``--dump-plan``
  document): same top-level keys and per-transfer fields, descriptor tables as
  base64 wire blobs, the per-rank ``layouts`` exactly as the reference's.

The transfers describe THIS design's data movement, derived from the device
plan (``GpuPlan``): there is no forwarder landing buffer, so

* dispatch ``node_transfers``: one per (source rank s, destination rank g),
  tokens ascending, sent once per rank (the per-rank dedup) from
  ``token/s`` straight into the token's primary row of ``activation/g`` (the
  row of its first k owned by g); ``local_edges`` per destination node: own
  tokens ``token/g -> activation/g`` and the receiver fan-out
  ``activation/g (primary) -> activation/g (duplicate)``;
* combine ``node_transfers``: one per (owner g, source s), every (t, k) row of
  ``act_out/g`` pulled into ``staging/s`` row ``local_rank(t)·K + k`` (the
  reference's staging index, planner.py:366 — here the pulled rows are
  reduced on arrival instead of being staged); ``local_edges``: own rows.
"""

from __future__ import annotations

import base64
import struct

import numpy as np

_HEADER = struct.Struct("<Q")


def descriptor_to_bytes(offsets, lengths) -> bytes:
    """Wire form of a descriptor list (descriptor.py:224-230)."""
    off = np.asarray(offsets, dtype=np.int64).reshape(-1)
    ln = np.asarray(lengths, dtype=np.int64).reshape(-1)
    if off.shape != ln.shape:
        raise ValueError("offsets and lengths must have the same length")
    if (off < 0).any() or (ln < 0).any():
        raise ValueError("descriptor offsets and lengths must be non-negative")
    table = np.empty((off.size, 2), dtype="<u8")
    table[:, 0] = off
    table[:, 1] = ln
    return _HEADER.pack(off.size) + table.tobytes()


def descriptor_from_bytes(blob: bytes) -> tuple[np.ndarray, np.ndarray]:
    """(offsets, lengths) from a wire blob (descriptor.py:232-241)."""
    if len(blob) < _HEADER.size:
        raise ValueError("descriptor blob too short for header")
    (n,) = _HEADER.unpack_from(blob)
    body = blob[_HEADER.size:]
    if len(body) != n * 16:
        raise ValueError(f"descriptor blob: expected {n} pairs, got {len(body)} bytes")
    table = np.frombuffer(body, dtype="<u8").reshape(n, 2)
    return table[:, 0].astype(np.int64), table[:, 1].astype(np.int64)


def _blob(buffer_id: str, offsets, tb: int) -> dict:
    offsets = np.asarray(offsets, dtype=np.int64)
    return {"buffer": buffer_id,
            "table": base64.b64encode(descriptor_to_bytes(offsets, np.full(offsets.size, tb))).decode("ascii")}


def _rows(plan):
    """All activation rows as parallel arrays (rank, row, token, k, source)."""
    g_l, r_l, t_l, k_l, s_l = [], [], [], [], []
    for g in sorted(plan.layouts):
        lay = plan.layouts[g]
        n = lay.num_rows
        g_l.append(np.full(n, g, dtype=np.int64))
        r_l.append(np.arange(n, dtype=np.int64))
        t_l.append(np.asarray(lay.token_ids, dtype=np.int64))
        k_l.append(np.asarray(lay.k_col, dtype=np.int64))
        s_l.append(np.asarray(lay.src_flat, dtype=np.int64))
    cat = lambda xs: np.concatenate(xs) if xs else np.zeros(0, dtype=np.int64)  # noqa: E731
    return cat(g_l), cat(r_l), cat(t_l), cat(k_l), cat(s_l)


def _local_rank(plan) -> np.ndarray:
    lr = np.full(plan.num_tokens, -1, dtype=np.int64)
    for s, ids in plan.local_tokens.items():
        lr[np.asarray(ids, dtype=np.int64)] = np.arange(len(ids), dtype=np.int64)
    return lr


def plan_to_json(plan, gpus_per_node: int = 1) -> dict:
    """The reference's ``plan_to_json`` document for a device plan (see module doc)."""
    tb, K = plan.token_bytes, plan.topk
    g, r, t, k, s = _rows(plan)
    lr = _local_rank(plan)
    node = lambda x: int(x) // gpus_per_node  # noqa: E731
    transfers, edges = [], {}
    if plan.direction == "dispatch":
        # primary row of (token, rank): the row of the token's first k owned by that rank
        order = np.lexsort((k, t, g))
        g_o, t_o, r_o, s_o = g[order], t[order], r[order], s[order]
        first = np.ones(order.size, dtype=bool)
        first[1:] = (g_o[1:] != g_o[:-1]) | (t_o[1:] != t_o[:-1])
        prim_row = np.maximum.accumulate(np.where(first, np.arange(order.size), 0))
        primary_of = r_o[prim_row]
        remote = first & (s_o != g_o)
        sel = np.flatnonzero(remote)
        key = np.lexsort((t_o[sel], g_o[sel], s_o[sel]))
        sel = sel[key]
        for src, dst in sorted({(int(a), int(b)) for a, b in zip(s_o[sel], g_o[sel])}):
            m = sel[(s_o[sel] == src) & (g_o[sel] == dst)]
            transfers.append({
                "src_flat": src, "dst_flat": dst, "dest_node": node(dst), "channel": ["group", 0],
                "bytes": int(m.size) * tb,
                "send": _blob(f"token/{src}", lr[t_o[m]] * tb, tb),
                "recv": _blob(f"activation/{dst}", r_o[m] * tb, tb),
            })
        for dst in sorted(plan.layouts):
            own = np.flatnonzero((g_o == dst) & (s_o == dst))
            own = own[np.argsort(r_o[own], kind="stable")]
            dup = np.flatnonzero((g_o == dst) & ~first & (s_o != dst))
            dup = dup[np.argsort(r_o[dup], kind="stable")]
            lst = edges.setdefault(str(node(dst)), [])
            if own.size:
                lst.append({"src_flat": dst, "dst_flat": dst, "bytes": int(own.size) * tb,
                            "send": _blob(f"token/{dst}", lr[t_o[own]] * tb, tb),
                            "recv": _blob(f"activation/{dst}", r_o[own] * tb, tb)})
            if dup.size:
                lst.append({"src_flat": dst, "dst_flat": dst, "bytes": int(dup.size) * tb,
                            "send": _blob(f"activation/{dst}", primary_of[dup] * tb, tb),
                            "recv": _blob(f"activation/{dst}", r_o[dup] * tb, tb)})
    elif plan.direction == "combine":
        for own_g in sorted(plan.layouts):
            for src in sorted(set(int(x) for x in s[g == own_g])):
                m = np.flatnonzero((g == own_g) & (s == src))
                m = m[np.lexsort((k[m], t[m]))]
                item = {"src_flat": own_g, "dst_flat": src, "bytes": int(m.size) * tb,
                        "send": _blob(f"act_out/{own_g}", r[m] * tb, tb),
                        "recv": _blob(f"staging/{src}", (lr[t[m]] * K + k[m]) * tb, tb)}
                if src == own_g:
                    edges.setdefault(str(node(own_g)), []).append(item)
                else:
                    transfers.append({**item, "dest_node": node(src), "channel": ["group", 0]})
    else:
        raise ValueError(f"unknown plan direction {plan.direction!r}")
    return {
        "direction": plan.direction,
        "token_bytes": tb,
        "num_tokens": plan.num_tokens,
        "topk": K,
        "groups": None if plan.groups is None else np.asarray(plan.groups).tolist(),
        "inter_bytes_total": int(plan.inter_bytes_total),
        "intra_bytes_total": int(plan.intra_bytes_total),
        "intra_gpu_bytes": int(plan.intra_gpu_bytes),
        "buffer_bytes": dict(sorted((str(a), int(b)) for a, b in plan.buffer_bytes.items())),
        "node_transfers": transfers,
        "local_edges": edges,
        "layouts": {
            str(gg): {
                "expert_ids": np.asarray(lay.expert_ids).tolist(),
                "token_ids": np.asarray(lay.token_ids).tolist(),
                "src_flat": np.asarray(lay.src_flat).tolist(),
                "k_col": np.asarray(lay.k_col).tolist(),
            }
            for gg, lay in sorted(plan.layouts.items())
        },
    }
