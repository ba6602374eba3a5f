"""ctypes bindings to the in-tree native libraries.

``engine()`` loads ``librpq_b200.so`` (the CUDA engine behind
include/rpq_b200.h).  There is no CPU fallback: if the library is missing or
cannot be loaded, every query raises.  ``datagen()`` loads the host-side
synthetic input generator.
"""

import ctypes
import os
import threading

from . import _build

RPQ_OK = 0
RPQ_EINVAL = 1
RPQ_ERANGE = 2
RPQ_ETIMEOUT = 3
RPQ_ECUDA = 4
RPQ_ENOMEM = 5
RPQ_ENOLABEL = 6

DIR_AUTO = 0
DIR_PUSH = 1
DIR_PULL = 2

STATS_LEVELS = 64
ABI_VERSION = 3  # include/rpq_b200.h RPQ_ABI_VERSION

# rpq_query_set_tuning keys (include/rpq_b200.h RPQ_TUNE_*)
TUNE_EMIT_MODE = 0
TUNE_EMIT_INLINE_MAX = 1
TUNE_TRACE = 2
TUNE_FLAGS = 3
TUNE_SMALL = 4
TUNE_DEFER = 5
TUNE_ZERO_COPY = 6

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_u64 = ctypes.c_uint64
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p
P_i32 = ctypes.POINTER(ctypes.c_int32)
P_i64 = ctypes.POINTER(ctypes.c_int64)
P_u8 = ctypes.POINTER(ctypes.c_uint8)
P_u32 = ctypes.POINTER(ctypes.c_uint32)
P_u64 = ctypes.POINTER(ctypes.c_uint64)


class RpqStats(ctypes.Structure):
    _fields_ = [
        ("status", c_i32),
        ("iterations", c_i32),
        ("levels", c_i32),
        ("grid", c_i32),
        ("te", c_i64),
        ("segments", c_i64),
        ("visited_pairs", c_i64),
        ("reach_count", c_i64),
        ("device_ms", ctypes.c_float),
        ("pull_levels", c_i32),
        ("level_new", c_i64 * STATS_LEVELS),
        ("level_edges", c_i64 * STATS_LEVELS),
        ("level_ns", c_i64 * STATS_LEVELS),
        ("work_ns", c_i64 * STATS_LEVELS),
        ("bar_ns", c_i64 * STATS_LEVELS),
        ("level_dir", ctypes.c_int8 * STATS_LEVELS),
        ("answer_list", c_i32),
        ("answer_words", c_i64),
    ]

    def to_dict(self):
        nlev = min(max(self.iterations, 0) + 1, STATS_LEVELS)
        return {
            "status": self.status,
            "iterations": self.iterations,
            "levels": self.levels,
            "grid": self.grid,
            "te": self.te,
            "segments": self.segments,
            "visited_pairs": self.visited_pairs,
            "reach_count": self.reach_count,
            "device_ms": self.device_ms,
            "pull_levels": self.pull_levels,
            "level_dir": list(self.level_dir[:nlev]),
            "level_us": [t / 1e3 for t in self.level_ns[:nlev]],
            "work_us": [t / 1e3 for t in self.work_ns[:nlev]],
            "bar_us": [t / 1e3 for t in self.bar_ns[:nlev]],
            "level_new": list(self.level_new[:nlev]),
            "level_edges": list(self.level_edges[:nlev]),
        }


BATCH = 64  # include/rpq_b200.h RPQ_BATCH


class RpqBatchStats(ctypes.Structure):
    _fields_ = [
        ("status", c_i32),
        ("nsrc", c_i32),
        ("levels", c_i32),
        ("grid", c_i32),
        ("te", c_i64),
        ("rows", c_i64),
        ("visited_pairs", c_i64),
        ("device_ms", ctypes.c_float),
        ("iterations", c_i32 * BATCH),
        ("reach_count", c_i64 * BATCH),
        ("level_items", c_i64 * STATS_LEVELS),
        ("level_new", c_i64 * STATS_LEVELS),
        ("level_ns", c_i64 * STATS_LEVELS),
        ("level_rows", c_i64 * STATS_LEVELS),
    ]

    def to_dict(self):
        nlev = min(max(self.levels, 0), STATS_LEVELS)
        return {
            "status": self.status,
            "nsrc": self.nsrc,
            "levels": self.levels,
            "grid": self.grid,
            "te": self.te,
            "rows": self.rows,
            "visited_pairs": self.visited_pairs,
            "device_ms": self.device_ms,
            "iterations": list(self.iterations[: self.nsrc]),
            "reach_count": list(self.reach_count[: self.nsrc]),
            "level_items": list(self.level_items[:nlev]),
            "level_new": list(self.level_new[:nlev]),
            "level_us": [t / 1e3 for t in self.level_ns[:nlev]],
            "level_rows": list(self.level_rows[:nlev]),
        }


# symbol -> (restype, argtypes); the complete C ABI of include/rpq_b200.h
ENGINE_SIGNATURES = {
    "rpq_abi_version": (c_i32, []),
    "rpq_checked_build": (c_i32, []),
    "rpq_last_error": (ctypes.c_char_p, []),
    "rpq_device_info": (c_i32, [c_i32, P_i32, P_i64, P_i64]),
    "rpq_graph_create": (c_i32, [c_i32, c_i32, c_i32, ctypes.POINTER(c_vp)]),
    "rpq_graph_set_label": (c_i32, [c_vp, c_i32, c_i64, P_i64, P_i64, c_i64, P_i64, P_i64]),
    "rpq_graph_set_label_i32": (c_i32, [c_vp, c_i32, c_i64, P_i32, P_i32, c_i64, P_i32, P_i32]),
    "rpq_graph_create_coo": (c_i32, [c_i32, c_i32, c_i64, P_i32, P_i32, P_i32, c_i32,
                                     ctypes.POINTER(c_vp)]),
    "rpq_graph_materialize_label": (c_i32, [c_vp, c_i32]),
    "rpq_graph_copy_label": (c_i32, [c_vp, c_i32, c_i32, P_u32, P_i32, c_i64, P_i64]),
    "rpq_graph_label_resident": (c_i32, [c_vp, c_i32]),
    "rpq_graph_device_bytes": (c_i64, [c_vp]),
    "rpq_graph_destroy": (c_i32, [c_vp]),
    "rpq_query_create": (c_i32, [c_vp, c_i32, c_i32, P_i32, P_i32, P_u8, P_i32, c_i32, P_i32,
                                 c_i32, P_i32, ctypes.POINTER(c_vp)]),
    "rpq_query_set_options": (c_i32, [c_vp, c_i32, c_i32, c_dbl]),
    "rpq_query_set_tuning": (c_i32, [c_vp, c_i32, c_dbl]),
    "rpq_query_run": (c_i32, [c_vp, c_i32, c_dbl, c_vp]),
    "rpq_query_wait": (c_i32, [c_vp, ctypes.POINTER(RpqStats)]),
    "rpq_query_reach_device": (c_i32, [c_vp, ctypes.POINTER(P_u8)]),
    "rpq_query_copy_reach": (c_i32, [c_vp, P_u8]),
    "rpq_query_copy_visited": (c_i32, [c_vp, P_u32, c_i64]),
    "rpq_query_step": (c_i32, [c_vp, P_u32, P_u32, c_i64, P_u32]),
    "rpq_query_set_output": (c_i32, [c_vp, c_i32]),
    "rpq_host_alloc": (c_i32, [c_i64, ctypes.POINTER(c_vp)]),
    "rpq_query_step_begin": (c_i32, [c_vp, c_vp]),
    "rpq_query_step_end": (c_i32, [c_vp, ctypes.POINTER(c_i64)]),
    "rpq_host_free": (c_i32, [c_vp]),
    "rpq_query_copy_reach_bits": (c_i32, [c_vp, P_u32, c_i64]),
    "rpq_query_io_bytes": (c_i32, [c_vp, P_i64, P_i64]),
    "rpq_query_destroy": (c_i32, [c_vp]),
    "rpq_query_row_words": (c_i32, [c_vp, P_i64]),
    "rpq_query_set_owned": (c_i32, [c_vp, c_i64, c_i64]),
    # (stats and answer buffers as void*: the per-query fast path passes raw addresses)
    "rpq_query_eval": (c_i32, [c_vp, c_i32, c_dbl, c_i32, c_i32, c_dbl, c_i32, c_vp, c_vp, c_i64]),
    "rpq_query_eval_list": (c_i32, [c_vp, c_i32, c_dbl, c_i32, c_i32, c_dbl, c_i32, c_vp, c_vp, c_i64]),
    "rpq_query_copy_trace": (c_i32, [c_vp, P_u64, c_i64, P_i32]),
    "rpq_query_step_device": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "rpq_query_run_batch": (c_i32, [c_vp, c_i32, P_i32, c_dbl, c_vp]),
    "rpq_query_wait_batch": (c_i32, [c_vp, ctypes.POINTER(RpqBatchStats)]),
    "rpq_query_copy_batch_bits": (c_i32, [c_vp, P_u32, c_i64]),
    "rpq_query_batch_bits_device": (c_i32, [c_vp, ctypes.POINTER(P_u32), P_i64]),
    "rpq_ssr": (c_i32, [c_vp, c_i32, c_i32, P_i32, P_i32, P_u8, P_i32, c_i32, P_i32, c_i32, P_i32,
                        c_i32, c_dbl, P_u8, ctypes.POINTER(RpqStats)]),
    "rpq_ssr_wide": (c_i32, [c_vp, c_i32, c_i32, P_i32, P_i32, P_u8, P_i32, c_i32, P_i32, c_i32, P_i32,
                             c_i32, c_dbl, P_u32, c_i64, ctypes.POINTER(RpqStats)]),
}

# table limits of the persistent kernel (csrc/ssr_kernel.cuh kMaxStates / kMaxGroups /
# kMaxSlots); automata beyond them run through rpq_ssr_wide
MAX_STATES = 256
MAX_GROUPS = 256
MAX_SLOTS = 128

DATAGEN_SIGNATURES = {
    "rpqgen_draw": (c_u64, [c_u64, c_u64, c_u64]),
    "rpqgen_zipf_thresholds": (None, [c_i32, c_dbl, P_u64]),
    "rpqgen_er": (c_i64, [c_i32, c_i64, c_i32, c_u64, P_i32, P_i32, P_i32]),
    "rpqgen_rmat": (c_i64, [c_i32, c_i64, c_dbl, c_dbl, c_dbl, c_i32, c_dbl, c_u64, P_i32, P_i32,
                            P_i32]),
    "rpqgen_chunglu": (c_i64, [c_i32, c_i64, c_dbl, c_i32, c_dbl, c_u64, P_i32, P_i32, P_i32]),
    "rpqgen_label_count": (c_i64, [c_i64, P_i32, c_i32]),
    "rpqgen_label_csr": (c_i64, [c_i32, c_i64, P_i32, P_i32, P_i32, c_i32, c_i32, P_i64, P_i64]),
    "rpqgen_out_degree": (None, [c_i32, c_i64, P_i32, P_i64]),
}

_lock = threading.Lock()
_engine = None
_datagen = None


class NativeLibraryMissing(RuntimeError):
    """The CUDA engine library is not built; there is no fallback path."""


def _bind(path, signatures):
    lib = ctypes.CDLL(path)
    for name, (res, args) in signatures.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def engine():
    """The loaded CUDA engine library (raises if it is not built)."""
    global _engine
    if _engine is None:
        with _lock:
            if _engine is None:
                # RPQ_ENGINE=checked: the bounds-checked build (tests/diagnostics)
                path = _build.CHECKED_SO if os.environ.get("RPQ_ENGINE") == "checked" else _build.ENGINE_SO
                path = os.environ.get("RPQ_ENGINE_SO", path)  # experiments: an alternative build
                if not os.path.exists(path):
                    raise NativeLibraryMissing(
                        f"{path} is not built; run "
                        "`python -m paper_2412_10287_b200._build` (there is no CPU fallback)"
                    )
                lib = _bind(path, ENGINE_SIGNATURES)
                if lib.rpq_abi_version() != ABI_VERSION:
                    raise NativeLibraryMissing("librpq_b200.so ABI version mismatch")
                _engine = lib
    return _engine


def datagen():
    global _datagen
    if _datagen is None:
        with _lock:
            if _datagen is None:
                if not os.path.exists(_build.DATAGEN_SO):
                    _build.build_datagen()
                _datagen = _bind(_build.DATAGEN_SO, DATAGEN_SIGNATURES)
    return _datagen


def last_error():
    msg = engine().rpq_last_error()
    return msg.decode() if msg else ""


def ptr(arr, ctype):
    """Pointer to a contiguous numpy array's data (None for empty arrays)."""
    if arr is None:
        return None
    return arr.ctypes.data_as(ctypes.POINTER(ctype))
