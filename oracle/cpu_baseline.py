"""CPU baseline = the oracle's restatement of the reference CPU path, timed.

TEST / BASELINE INFRASTRUCTURE ONLY: used by bench.py's ``cpu_baseline``
leg and ``--impl reference`` arm, never by the product path.  Same arithmetic
as ``shuffle_oracle`` (reference planner.py:138-159 layout, engine.py:266-276
row moves, engine.py:313-338 f64 k-ascending reduction), chunked over tokens
and run on a thread pool so the baseline uses every host core numpy can use
(numpy releases the GIL inside large copies and ufuncs).  Chunking by token
does not change any per-token result.
"""

from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import shuffle_oracle as O


def _chunks(n: int, parts: int):
    step = max(1, -(-n // max(1, parts)))
    return [(lo, min(n, lo + step)) for lo in range(0, n, step)]


def shuffle_times(experts, weights, source, owner, num_ranks, payload, dtype="bf16", threads=None):
    """(plan_s, dispatch_s, combine_s) of one full exchange on the host."""
    threads = threads or os.cpu_count() or 1
    pool = ThreadPoolExecutor(threads)
    try:
        t0 = time.perf_counter()
        layouts, row_of = O.activation_layouts(experts, source, owner, num_ranks)
        t1 = time.perf_counter()
        acts = {g: np.empty((lay.num_rows, payload.shape[1]), dtype=np.uint8) for g, lay in layouts.items()}

        def disp(g, lo, hi):
            np.take(payload, layouts[g].token_ids[lo:hi], axis=0, out=acts[g][lo:hi])

        list(pool.map(lambda a: disp(*a), [(g, lo, hi) for g in layouts for lo, hi in
                                            _chunks(layouts[g].num_rows, threads)]))
        t2 = time.perf_counter()
        ids = [np.flatnonzero(source == s) for s in range(num_ranks)]
        outs = {s: np.empty((ids[s].size, payload.shape[1]), dtype=np.uint8) for s in range(num_ranks)}

        def comb(s, lo, hi):
            outs[s][lo:hi] = O.combine(acts, row_of, experts, weights, owner, ids[s][lo:hi], dtype)

        list(pool.map(lambda a: comb(*a), [(s, lo, hi) for s in range(num_ranks) for lo, hi in
                                            _chunks(ids[s].size, threads)]))
        t3 = time.perf_counter()
    finally:
        pool.shutdown()
    return t1 - t0, t2 - t1, t3 - t2, threads
