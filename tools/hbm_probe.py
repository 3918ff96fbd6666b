"""HBM ceilings by access mix on this B200 (what bounds a write-heavy mover).

    python tools/hbm_probe.py

Times (CUDA events, best of 10, 2 GiB buffers) a read+write copy, a write-only
fill and a read-only reduction, plus the engine's own 16-byte warp copy
(fs_probe_copy).  The DeepSeek-V3 single-GPU dispatch is 1 read : 8 writes,
so the write-only figure is its ceiling.
"""

import json
import sys
from ctypes import c_void_p
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def best(fn, nbytes, reps=10):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    fn()
    torch.cuda.synchronize()
    t = []
    for _ in range(reps):
        ev[0].record()
        fn()
        ev[1].record()
        ev[1].synchronize()
        t.append(ev[0].elapsed_time(ev[1]) * 1e-3)
    return nbytes / min(t) / 1e9


def main():
    from paper_2512_22036_b200 import _lib

    n = 2 << 30
    a = torch.empty(n, dtype=torch.uint8, device="cuda").fill_(1)
    b = torch.empty(n, dtype=torch.uint8, device="cuda")
    out = {
        "copy_rw_gbs": best(lambda: b.copy_(a), 2 * n),
        "fill_w_gbs": best(lambda: b.fill_(3), n),
        "sum_r_gbs": best(lambda: a.view(torch.int64).sum(), n),
    }
    lib = _lib.load()
    st = c_void_p(torch.cuda.current_stream().cuda_stream)
    for ctas in (148 * 4, 148 * 8):
        out[f"fs_probe_copy_{ctas}_gbs"] = best(
            lambda: _lib.check(lib.fs_probe_copy(0, c_void_p(b.data_ptr()), c_void_p(a.data_ptr()), n, ctas, st)),
            2 * n)
    for ctas in (148 * 4, 148 * 8):
        out[f"fs_probe_fill_{ctas}_gbs"] = best(
            lambda: _lib.check(lib.fs_probe_copy(0, c_void_p(b.data_ptr()), c_void_p(0), n, ctas, st)), n)
    # the P=1 dispatch's pattern: 4096 rows of 14336 B, each written to 8 of
    # 32768 destination rows in a random order (read 59 MB, write 470 MB)
    rows, fan, rb = 4096, 8, 14336
    src = torch.empty(rows * rb, dtype=torch.uint8, device="cuda").fill_(1)
    dst = torch.empty(rows * fan * rb, dtype=torch.uint8, device="cuda")
    perm = torch.randperm(rows * fan, device="cuda").to(torch.int32)
    for ctas in (148 * 3, 148 * 6):
        for ro in (0, 1):
            out[f"fs_probe_scatter_{'w' if ro else 'rw'}_{ctas}_gbs"] = best(
                lambda: _lib.check(lib.fs_probe_scatter(0, c_void_p(dst.data_ptr()),
                                                        c_void_p(0 if ro else src.data_ptr()),
                                                        c_void_p(perm.data_ptr()), rows, fan, rb, ctas, st)),
                rows * fan * rb + (0 if ro else rows * rb))
    print(json.dumps({k: round(v, 1) for k, v in out.items()}))


if __name__ == "__main__":
    main()
