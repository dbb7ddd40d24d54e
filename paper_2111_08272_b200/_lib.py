"""ctypes declarations of libpropring.so (include/propring.h).  Argument marshalling only.

The library is built in-tree (paper_2111_08272_b200/libpropring.so, see build.py).  There is no
fallback: if the shared object is missing, importing the package raises.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# PROPRING_LIB: another build of this same library (tools/variants.sh compiles A/B variants for profiling)
LIB_PATH = os.environ.get("PROPRING_LIB") or os.path.join(HERE, "libpropring.so")

PR_MAX_RANKS = 64
PR_GATHER_MAX_CHANNELS = 16

c_i32, c_i64, c_u64, c_vp, c_dbl, c_sz = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p,
                                          ctypes.c_double, ctypes.c_size_t)


class AllocView(ctypes.Structure):
    _fields_ = [("N", c_i64), ("P", c_i32), ("frozen", c_i32), ("C", c_i64), ("g", c_i64), ("floor", c_i64),
                ("B", c_i64), ("S", c_i64), ("epoch", c_i64), ("hist_len", c_i64),
                ("w", c_i64 * PR_MAX_RANKS), ("n", c_i64 * PR_MAX_RANKS), ("len", c_i64 * PR_MAX_RANKS),
                ("off", c_i64 * PR_MAX_RANKS)]


class AllocPolicy(ctypes.Structure):
    _fields_ = [("window", c_i32), ("never_freeze", c_i32), ("tol", c_i64), ("ema_alpha", c_dbl),
                ("model", c_i32), ("fit_window", c_i32)]


class GatherOp(ctypes.Structure):
    _fields_ = [("op", c_i32), ("channels", c_i32), ("plane", c_i64),
                ("scale", ctypes.c_float * PR_GATHER_MAX_CHANNELS), ("shift", ctypes.c_float * PR_GATHER_MAX_CHANNELS),
                ("impl", c_i32), ("layout", c_i32)]


class CommConfig(ctypes.Structure):
    _fields_ = [("channels", c_i32), ("slots", c_i32), ("threads", c_i32), ("flags", c_i32),
                ("slot_bytes", c_i64), ("watchdog_ns", c_i64), ("stages", c_i32), ("tile_bytes", c_i32),
                ("algo", c_i32), ("ts_slots", c_i32), ("ts_slot_bytes", c_i64), ("ts_max_bytes", c_i64),
                ("ll_max_bytes", c_i64), ("os_max_bytes", c_i64), ("min_slice_bytes", c_i64)]


EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int, c_vp, c_vp, c_sz, c_vp)

# name -> (restype, argtypes); every `pr_*` declaration of include/propring.h
SIGNATURES = {
    "pr_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "pr_version": (ctypes.c_int, []),
    "pr_alloc_init": (ctypes.c_int, [ctypes.POINTER(c_vp), c_i64, c_i32, ctypes.POINTER(c_dbl), c_i64, c_i64, c_i64]),
    "pr_alloc_set_policy": (ctypes.c_int, [c_vp, ctypes.POINTER(AllocPolicy)]),
    "pr_alloc_update": (ctypes.c_int, [c_vp, ctypes.POINTER(c_dbl), ctypes.POINTER(c_i32)]),
    "pr_alloc_query": (ctypes.c_int, [c_vp, ctypes.POINTER(AllocView)]),
    "pr_alloc_history": (ctypes.c_int, [c_vp, c_i64, ctypes.POINTER(c_i64)]),
    "pr_alloc_save": (ctypes.c_int, [c_vp, c_vp, c_sz, ctypes.POINTER(c_sz)]),
    "pr_alloc_load": (ctypes.c_int, [ctypes.POINTER(c_vp), c_vp, c_sz]),
    "pr_alloc_destroy": (None, [c_vp]),
    "pr_shard_indices": (ctypes.c_int, [c_vp, c_i32, c_i64, c_u64, c_vp, c_i64, c_vp]),
    "pr_shard_steps": (ctypes.c_int, [c_vp, c_i32, c_i64, c_u64, c_i64, c_i64, c_vp, c_i64, c_vp]),
    "pr_permute": (ctypes.c_int, [c_i64, c_u64, c_i64, c_i64, c_i64, c_vp, c_vp]),
    "pr_gather_rows": (ctypes.c_int, [c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, ctypes.POINTER(GatherOp), c_vp, c_vp, c_vp]),
    "pr_spin": (ctypes.c_int, [c_i64, c_vp]),
    "pr_stamp": (ctypes.c_int, [c_vp, c_i64, c_vp]),
    "pr_stamp_seconds": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp]),
    "pr_sgd_update": (ctypes.c_int, [c_vp, c_vp, c_i64, c_dbl, c_dbl, c_i32, c_vp]),
    "pr_comm_init": (ctypes.c_int, [ctypes.POINTER(c_vp), c_i32, c_i32, c_i32, EXCHANGE_FN, c_vp,
                                    ctypes.POINTER(CommConfig)]),
    "pr_comm_init_local": (ctypes.c_int, [ctypes.POINTER(c_vp), c_i32, c_i32, ctypes.POINTER(CommConfig)]),
    "pr_comm_register": (ctypes.c_int, [c_vp, c_vp, c_sz]),
    "pr_comm_alloc": (ctypes.c_int, [c_vp, c_sz, ctypes.POINTER(c_vp)]),
    "pr_weighted_allreduce": (ctypes.c_int, [c_vp, c_vp, c_i64, c_i32, c_i64, c_vp]),
    "pr_weighted_allreduce_local": (ctypes.c_int, [ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), c_i64, c_i32,
                                                   ctypes.POINTER(c_i64), c_vp]),
    "pr_weighted_allreduce_sgd": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, c_i64, c_dbl, c_dbl, c_i32, c_vp]),
    "pr_weighted_allreduce_sgd_local": (ctypes.c_int, [ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), ctypes.POINTER(c_vp),
                                                       c_i64, ctypes.POINTER(c_i64), c_dbl, c_dbl, c_i32, c_vp]),
    "pr_comm_allgather_f64": (ctypes.c_int, [c_vp, c_dbl, ctypes.POINTER(c_dbl), c_vp]),
    "pr_comm_allgather_f64_async": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "pr_comm_nvls_alloc": (ctypes.c_int, [c_vp, ctypes.c_size_t, ctypes.POINTER(c_vp)]),
    "pr_comm_status": (ctypes.c_int, [c_vp]),
    "pr_comm_timestamps": (ctypes.c_int, [c_vp, ctypes.POINTER(c_i64)]),
    "pr_comm_rank": (ctypes.c_int, [c_vp, ctypes.POINTER(c_i32), ctypes.POINTER(c_i32)]),
    "pr_comm_destroy": (None, [c_vp]),
    "pr_test_philox": (ctypes.c_int, [c_vp, c_i64, c_u64, c_i32, c_vp, c_vp]),
}


def load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python paper_2111_08272_b200/build.py` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        if os.environ.get("PROPRING_LIB") and not hasattr(lib, name):
            continue     # an older A/B build (tools/variants.sh) may predate an entry point
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    lib.pr_last_cuda_error.restype = ctypes.c_char_p
    lib.pr_last_cuda_error.argtypes = []
    return lib


LIB = load()
