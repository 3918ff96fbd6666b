"""CPU oracle for the Fusco shuffle path — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference package's (``shuffleforge``) CPU
algorithm for the hot path, used only by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU-baseline leg as the *checker*.  The product path
(``paper_2512_22036_b200``) never imports this module.

Parity is pinned: ``tests/test_oracle.py`` checks every function below
against golden vectors produced by the reference itself
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``) and, when
``/root/reference`` is present, against the live reference on random cases.

Functions and the reference lines they restate (paths relative to the
reference ``pkg/src/shuffleforge/``):

* ``first_mask``            routing.py:86-98   derive_token_node
* ``activation_layouts``    planner.py:138-159 _activation_layouts (+ row_of)
* ``dispatch_loads``        planner.py:178-196
* ``naive_remote_rows``     planner.py:199-208
* ``dispatch``              engine.py:266-276 (apply_node_level +
                            apply_expert_level, dispatch plan): activation row
                            r of rank g holds the payload of layouts[g].token_ids[r]
                            (the property test_engine.py:185-195 asserts)
* ``combine``               engine.py:266-276 (combine plan) + 313-338
                            (_reduce_one: f64 accumulate, k ascending, one
                            rounding to the payload dtype)
* ``scaled_expert``         engine.py:283-292
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


# ---------------------------------------------------------------------------
# bf16 helpers (numpy has no bfloat16: bf16 values travel as uint16 bits)


def bf16_to_f32(u16: np.ndarray) -> np.ndarray:
    return (np.asarray(u16, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even f32 -> bf16 bits (finite inputs)."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = b + 0x7FFF + ((b >> 16) & 1)
    return (b >> 16).astype(np.uint16)


def f64_to_bf16(x: np.ndarray) -> np.ndarray:
    """Single round-to-nearest-even f64 -> bf16 bits (what __double2bfloat16
    does).  Exact for values in the f32 normal range; values below it fall
    back to f64->f32->bf16 (documented double rounding, never hit by the
    standard-normal payloads the tests use)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    b = x.view(np.uint64)
    r = b + np.uint64((1 << 44) - 1) + ((b >> np.uint64(45)) & np.uint64(1))
    r &= ~np.uint64((1 << 45) - 1)
    out = f32_to_bf16(r.view(np.float64).astype(np.float32))
    tiny = np.abs(x) < np.finfo(np.float32).tiny
    if tiny.any():
        out[tiny] = f32_to_bf16(x[tiny].astype(np.float32))
    return out


# ---------------------------------------------------------------------------
# planner


def first_mask(experts: np.ndarray, owner: np.ndarray, gpus_per_node: int = 1) -> np.ndarray:
    """first_mask[t,k]: node of expert k not seen earlier in row t."""
    nodes = owner[experts] // gpus_per_node
    out = np.ones(nodes.shape, dtype=bool)
    for k in range(1, nodes.shape[1]):
        out[:, k] = (nodes[:, :k] != nodes[:, k : k + 1]).all(axis=1)
    return out


@dataclass
class Layout:
    expert_ids: np.ndarray
    token_ids: np.ndarray
    src: np.ndarray
    k_col: np.ndarray

    @property
    def num_rows(self) -> int:
        return int(self.token_ids.size)


def activation_layouts(experts: np.ndarray, source: np.ndarray, owner: np.ndarray, num_ranks: int):
    """Per rank: rows sorted by (expert, source, token); plus row_of[t,k]."""
    own = owner[experts]
    row_of = np.full(experts.shape, -1, dtype=np.int64)
    layouts = {}
    for g in range(num_ranks):
        ts, ks = np.nonzero(own == g)
        es = experts[ts, ks]
        order = np.lexsort((ts, source[ts], es))  # last key is primary
        ts, ks, es = ts[order], ks[order], es[order]
        row_of[ts, ks] = np.arange(ts.size)
        layouts[g] = Layout(es, ts, source[ts], ks)
    return layouts, row_of


def dispatch_loads(experts, source, owner, num_ranks, token_bytes, gpus_per_node=1) -> np.ndarray:
    """Per-source deduplicated remote send bytes: Σ_t |distinct remote nodes|·tb."""
    nodes = owner[experts] // gpus_per_node
    remote_first = first_mask(experts, owner, gpus_per_node) & (nodes != (source // gpus_per_node)[:, None])
    return np.bincount(source, weights=remote_first.sum(axis=1), minlength=num_ranks).astype(np.int64) * token_bytes


def naive_remote_rows(experts, source, owner, gpus_per_node=1) -> int:
    return int((owner[experts] // gpus_per_node != (source // gpus_per_node)[:, None]).sum())


def rank_dedup_rows(experts, source, owner) -> np.ndarray:
    """Per source rank: Σ_t |distinct destination ranks ≠ source| (one box)."""
    return dispatch_loads(experts, source, owner, int(source.max(initial=0)) + 1, 1, 1)


# ---------------------------------------------------------------------------
# executors


def dispatch(payloads: np.ndarray, layouts: dict) -> dict:
    """activation/g = payload rows in layout order (bytes, any dtype)."""
    return {g: payloads[lay.token_ids] for g, lay in layouts.items()}


def identity_expert(act_f32: np.ndarray, expert_ids: np.ndarray) -> np.ndarray:
    return act_f32


def scaled_expert(act_f32: np.ndarray, expert_ids: np.ndarray) -> np.ndarray:
    e = expert_ids.astype(np.float32)[:, None]
    return act_f32 * (e + 2) + e


def run_experts(activations: dict, layouts: dict, fn, dtype: str = "f32") -> dict:
    out = {}
    for g, act in activations.items():
        vals = decode(act, dtype)
        y = np.ascontiguousarray(fn(vals, layouts[g].expert_ids), dtype=np.float32)
        out[g] = encode(y, dtype)
    return out


def decode(rows_u8: np.ndarray, dtype: str) -> np.ndarray:
    """[n, token_bytes] uint8 rows -> [n, width] float32 values."""
    rows = np.ascontiguousarray(rows_u8, dtype=np.uint8)
    if dtype == "f32":
        return rows.view(np.float32)
    return bf16_to_f32(rows.view(np.uint16))


def encode(vals: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == "f32":
        return np.ascontiguousarray(vals, dtype=np.float32).view(np.uint8)
    return np.ascontiguousarray(f32_to_bf16(vals)).view(np.uint8)


def combine(act_out: dict, row_of: np.ndarray, experts: np.ndarray, weights: np.ndarray,
            owner: np.ndarray, token_ids: np.ndarray, dtype: str = "f32") -> np.ndarray:
    """Outputs of one source's tokens ``token_ids``: Σ_k w·row, f64, k ascending."""
    n = token_ids.size
    token_bytes = next(iter(act_out.values())).shape[-1]
    if n == 0:
        return np.zeros((0, token_bytes), dtype=np.uint8)

    def rows_of(k):
        g = owner[experts[token_ids, k]]
        r = row_of[token_ids, k]
        rows = np.empty((n, token_bytes), dtype=np.uint8)
        for gg in np.unique(g):
            sel = np.flatnonzero(g == gg)
            rows[sel] = act_out[int(gg)][r[sel]]
        return rows

    return reduce_rows(rows_of, weights[token_ids], dtype)


def reduce_rows(rows_of, weights: np.ndarray, dtype: str = "f32") -> np.ndarray:
    """engine.py:313-331 _reduce_one: out = Σ_k f64(w[:,k])·f64(row_k), k
    ascending, one final rounding to the payload dtype.  ``rows_of(k)`` gives
    the [n, token_bytes] staged rows of column k (what the combine plan
    delivers to the staging buffer)."""
    acc = None
    for k in range(weights.shape[1]):
        rows = decode(rows_of(k), dtype).astype(np.float64)
        if acc is None:
            acc = np.zeros_like(rows)
        acc += weights[:, k][:, None] * rows
    if dtype == "f32":
        return acc.astype(np.float32).view(np.uint8)
    return np.ascontiguousarray(f64_to_bf16(acc)).view(np.uint8)


def exchange(experts, weights, source, owner, num_ranks, payloads, expert_fn=identity_expert, dtype="f32",
             gpus_per_node: int = 1) -> dict:
    """Whole reference pipeline for one routing; returns every checked artefact."""
    layouts, row_of = activation_layouts(experts, source, owner, num_ranks)
    acts = dispatch(payloads, layouts)
    outs_act = acts if expert_fn is identity_expert else run_experts(acts, layouts, expert_fn, dtype)
    outputs = {}
    for s in range(num_ranks):
        ids = np.flatnonzero(source == s)
        outputs[s] = combine(outs_act, row_of, experts, weights, owner, ids, dtype)
    return {
        "layouts": layouts,
        "row_of": row_of,
        "first_mask": first_mask(experts, owner, gpus_per_node),
        "loads": dispatch_loads(experts, source, owner, num_ranks, payloads.shape[1], gpus_per_node),
        "activations": acts,
        "outputs": outputs,
    }
