"""ctypes binding of libfusco.so (the C ABI in include/fusco.h).

There is no fallback: if the library is missing or fails to load, every
entry point raises.  Error codes map to exceptions the way the reference
raises them: FS_EINVAL / FS_ERANGE -> ValueError (reference validation
errors, e.g. descriptor.py:107-114, routing.py:36-67), the rest ->
RuntimeError.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_int, c_longlong, c_size_t, c_uint, c_void_p
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libfusco.so"
HEADER = Path(__file__).resolve().parent.parent / "include" / "fusco.h"

FS_ABI_VERSION = ABI_VERSION = 2
FS_OK, FS_EINVAL, FS_ECUDA, FS_ETIMEOUT, FS_ERANGE = 0, -1, -2, -3, -4
FS_PHASE_LOCAL, FS_PHASE_REMOTE, FS_PHASE_ALL = 1, 2, 3
FS_DTYPE_F32, FS_DTYPE_BF16 = 0, 1
FS_SRC_ACT, FS_SRC_ACT_OUT = 0, 1
FS_ACC_F32, FS_ACC_F64 = 0, 1
FS_NSTATS = 8
FS_MAX_RANKS = 32
STAT_ROWS, STAT_DEDUP_SEND, STAT_NAIVE_SEND, STAT_LOCAL_ROWS, STAT_NODE_DEDUP = 0, 1, 2, 3, 4

# name -> (restype, argtypes)
SIGNATURES = {
    "fs_abi_version": (c_int, []),
    "fs_last_error": (c_char_p, []),
    "fs_region_bytes": (c_int, [c_int, c_int, c_int, c_int, c_int, c_longlong, c_int, POINTER(c_size_t)]),
    "fs_sym_alloc": (c_int, [c_int, c_size_t, POINTER(c_void_p)]),
    "fs_sym_free": (c_int, [c_int, c_void_p]),
    "fs_ipc_handle": (c_int, [c_int, c_void_p, c_void_p]),
    "fs_ipc_open": (c_int, [c_int, c_void_p, POINTER(c_void_p)]),
    "fs_ipc_close": (c_int, [c_int, c_void_p]),
    "fs_enable_peer_access": (c_int, [c_int, c_int]),
    "fs_create": (
        c_int,
        [c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_longlong, c_int, c_void_p, c_void_p, c_void_p,
         c_int, c_int, POINTER(c_void_p)],
    ),
    "fs_destroy": (c_int, [c_void_p]),
    "fs_num_local_experts": (c_int, [c_void_p, POINTER(c_int)]),
    "fs_grid_ctas": (c_int, [c_void_p, POINTER(c_int)]),
    "fs_buffer_ptr": (c_int, [c_void_p, c_int, POINTER(c_void_p)]),
    "fs_max_rows": (c_longlong, [c_void_p]),
    "fs_epoch": (c_uint, [c_void_p]),
    "fs_set_nodedup": (c_int, [c_void_p, c_int]),
    "fs_set_balance": (c_int, [c_void_p, c_int]),
    "fs_layout": (
        c_int,
        [c_void_p, c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
         c_int, c_void_p],
    ),
    "fs_dispatch": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_int, c_int, c_void_p]),
    "fs_dispatch_w": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_int, c_int, c_int, c_void_p]),
    "fs_combine": (
        c_int,
        [c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_int, c_int, c_void_p, c_int, c_int, c_int,
         c_int, c_void_p],
    ),
    "fs_check": (c_int, [c_void_p, c_void_p]),
    "fs_trace": (c_int, [c_void_p, c_void_p, c_void_p]),
    "fs_probe_a2a": (c_int, [c_int, c_void_p, c_void_p, c_int, c_size_t, c_int, c_int, c_void_p]),
    "fs_probe_copy": (c_int, [c_int, c_void_p, c_void_p, c_size_t, c_int, c_void_p]),
    "fs_probe_scatter": (c_int, [c_int, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_void_p]),
}

_lib = None


class FuscoError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"libfusco error {code}: {msg}")
        self.code = code


class FuscoValueError(ValueError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def load(path: str | os.PathLike | None = None) -> ctypes.CDLL:
    """Load libfusco.so (built by ``paper_2512_22036_b200.build``)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    # FUSCO_LIB: an alternative build of the same ABI (compile-time experiments)
    p = Path(path) if path is not None else Path(os.environ.get("FUSCO_LIB", LIB_PATH))
    if not p.exists():
        raise FuscoError(
            FS_ECUDA,
            f"{p} not found: build the CUDA extension first "
            "(python -c 'import __graft_entry__; __graft_entry__.build()')",
        )
    lib = ctypes.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.fs_abi_version() != ABI_VERSION:
        raise FuscoError(FS_ECUDA, "libfusco ABI version mismatch")
    if path is None:
        _lib = lib
    return lib


def check(rc: int) -> None:
    if rc == FS_OK:
        return
    msg = load().fs_last_error().decode(errors="replace")
    if rc in (FS_EINVAL, FS_ERANGE):
        raise FuscoValueError(rc, msg)
    raise FuscoError(rc, msg)


def call(name: str, *args) -> int:
    rc = getattr(load(), name)(*args)
    check(rc)
    return rc


def ptr(t) -> c_void_p:
    """Device pointer of a torch tensor (or None -> NULL)."""
    return c_void_p(0 if t is None else t.data_ptr())


def stream_ptr(stream=None) -> c_void_p:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return c_void_p(s.cuda_stream)
