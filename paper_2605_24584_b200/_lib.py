"""ctypes loader for the in-tree CUDA library (liblaplex_b200.so).

There is no CPU fallback: if the library is missing this raises immediately,
so a GPU test can never pass on a silent eager path.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
# LAPLEX_LIB: load an alternative in-tree build (diagnostic sweeps, tools/)
LIB_PATH = os.environ.get("LAPLEX_LIB") or os.path.join(HERE, "liblaplex_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "laplex_c.h")

_lib = None

vp = C.c_void_p
sz = C.c_size_t
u64p = C.POINTER(C.c_uint64)

_SIGS = {
    "laplex_abi_version": (C.c_int, []),
    "laplex_last_error": (C.c_char_p, []),
    "laplex_kernel_launches": (C.c_uint64, []),
    "laplex_profile_enable": (C.c_int, [C.c_int]),
    "laplex_profile_dump": (C.c_int, [C.c_char_p, sz]),
    "laplex_plan_create": (C.c_int, [C.c_int, vp, sz, vp, sz, C.c_double, vp, vp, C.POINTER(vp)]),
    "laplex_plan_create_dev": (C.c_int, [C.c_int, vp, sz, vp, sz, C.c_double, vp, vp, vp, C.POINTER(vp)]),
    "laplex_plan_create_dev_async": (C.c_int, [C.c_int, vp, sz, vp, sz, C.c_double, vp, vp, vp, C.POINTER(vp)]),
    "laplex_plan_check": (C.c_int, [vp]),
    "laplex_pool_trim": (C.c_int, []),
    "laplex_gram_apply": (C.c_int, [vp, vp, sz, sz, vp]),
    "laplex_gram_apply_dev": (C.c_int, [vp, vp, sz, vp, vp]),
    "laplex_plan_retain": (C.c_int, [vp]),
    "laplex_plan_release": (C.c_int, [vp]),
    "laplex_plan_transposed": (C.c_int, [vp, C.POINTER(vp)]),
    "laplex_plan_shape": (C.c_int, [vp, C.POINTER(sz), C.POINTER(sz), C.POINTER(C.c_double), C.POINTER(C.c_int),
                                    C.POINTER(C.c_int)]),
    "laplex_plan_sorted": (C.c_int, [vp, C.c_int, vp, vp, vp]),
    "laplex_plan_ranks": (C.c_int, [vp, C.c_int, C.c_int, vp]),
    "laplex_apply": (C.c_int, [vp, C.c_uint, vp, sz, sz, vp]),
    "laplex_apply_dev": (C.c_int, [vp, C.c_uint, vp, sz, vp, vp]),
    "laplex_backward": (C.c_int, [vp, C.c_uint, vp, sz, sz, vp, sz, vp, vp, vp, vp, vp]),
    "laplex_backward_dev": (C.c_int, [vp, C.c_uint, vp, vp, sz, vp, vp, vp, vp, vp, vp]),
    "laplex_gram": (C.c_int, [vp, C.c_uint, vp, sz, vp]),
    "laplex_gram_dev": (C.c_int, [vp, C.c_uint, vp, vp, vp]),
    "laplex_gram_vjp_weights": (C.c_int, [vp, vp, sz, vp, sz, sz, vp]),
    "laplex_sort": (C.c_int, [C.c_int, vp, sz, vp, vp, vp]),
    "laplex_sort_dev": (C.c_int, [C.c_int, vp, sz, vp, vp, vp, vp, vp]),
    "laplex_scan_dev": (C.c_int, [C.c_int, vp, sz, vp, vp, vp, vp]),
    "laplex_gram_vjp_weights_dev": (C.c_int, [vp, vp, vp, vp]),
    "laplex_shard_partition_dev": (C.c_int, [C.c_int, vp, sz, C.c_double, vp, C.c_int, vp, vp, vp]),
    "laplex_gather_dev": (C.c_int, [C.c_int, vp, sz, vp, sz, sz, vp, vp]),
    "laplex_scatter_dev": (C.c_int, [C.c_int, vp, vp, sz, sz, vp, sz, vp]),
    "laplex_shard_plan_create_dev": (C.c_int, [C.c_int, vp, sz, vp, sz, C.c_double, vp, vp, vp, C.POINTER(vp)]),
    "laplex_shard_totals_count": (C.c_int, [vp, C.c_uint, C.c_int, sz, C.POINTER(sz)]),
    "laplex_shard_apply_begin": (C.c_int, [vp, C.c_uint, vp, sz, vp, C.POINTER(vp), vp]),
    "laplex_shard_apply_end": (C.c_int, [vp, vp, vp, vp]),
    "laplex_shard_backward_begin": (C.c_int, [vp, C.c_uint, vp, vp, sz, vp, C.POINTER(vp), vp]),
    "laplex_shard_backward_end": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp]),
    "laplex_work_release": (C.c_int, [vp]),
    "laplex_nccl_unique_id": (C.c_int, [vp]),
    "laplex_comm_init_nccl": (C.c_int, [vp, C.c_int, C.c_int, C.POINTER(vp)]),
    "laplex_comm_init_local": (C.c_int, [C.c_uint64, C.c_int, C.c_int, C.POINTER(vp)]),
    "laplex_comm_destroy": (C.c_int, [vp]),
    "laplex_sharded_create_dev": (C.c_int, [vp, C.c_int, vp, sz, vp, sz, C.c_double, vp, C.POINTER(vp)]),
    "laplex_sharded_shape": (C.c_int, [vp, C.POINTER(sz), C.POINTER(sz)]),
    "laplex_sharded_apply_dev": (C.c_int, [vp, vp, sz, vp, vp]),
    "laplex_sharded_backward_dev": (C.c_int, [vp, C.c_uint, vp, vp, sz, vp, vp, vp, vp]),
    "laplex_sharded_release": (C.c_int, [vp]),
    "laplex_replica_backward_dev": (C.c_int, [vp, vp, C.c_uint, vp, vp, sz, vp, vp, vp, vp, vp, vp]),
    "laplex_scan": (C.c_int, [C.c_int, vp, sz, vp, vp, vp]),
}


def header_symbols() -> list[str]:
    """Every function declared in include/laplex_c.h."""
    with open(HEADER) as f:
        text = f.read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|uint64_t)\s+(laplex_\w+)\s*\(", text, re.M)))


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(the CUDA library is required; there is no CPU fallback)")
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib
