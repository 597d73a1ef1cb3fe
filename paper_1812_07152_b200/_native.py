"""ctypes bindings of the two native libraries of the package.

* ``libhmxg.so`` — the sm_100a evaluator behind the C-ABI of ``include/hmxg.h``.
* ``libhmxb.so`` — the multi-threaded host instance builder of ``include/hmxb.h``.

Both are built in-tree by ``__graft_entry__.build()``. There is no fallback: if a
library is missing or fails to load, every entry point raises ``NativeLibraryError``.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
HMXG_PATH = os.environ.get("HMXG_LIBRARY") or os.path.join(_HERE, "libhmxg.so")  # override: A/B builds
HMXB_PATH = os.path.join(_HERE, "libhmxb.so")

HMXG_OK, HMXG_EINVAL, HMXG_ECUDA, HMXG_ENOMEM, HMXG_ECOMM, HMXG_EIO, HMXG_EGUARD = 0, 1, 2, 3, 4, 5, 6
HMXG_KERNEL_GAUSSIAN, HMXG_KERNEL_EXPONENTIAL, HMXG_KERNEL_INVDIST = 0, 1, 2
HMXG_ERR_DENSE, HMXG_ERR_SAMPLED = 0, 1
HMXG_NO_NODE = 0xFFFFFFFF
HMXG_F_DEVICE_PTRS = 0x1
HMXG_F_NO_SYNC = 0x2
HMXG_F_TIME_PHASES = 0x4
HMXG_F_NO_GRAPH = 0x8
HMXG_F_LEVEL_LAUNCHES = 0x10
PHASE_KINDS = {0: "gather", 1: "upward", 2: "far+downward", 3: "near+leaf", 4: "scatter", 5: "dag", 6: "near",
               7: "near-gen"}
HMXG_UPLOAD_NEAR_ON_THE_FLY = 1

_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_f64p = C.POINTER(C.c_double)


class NativeLibraryError(RuntimeError):
    """A native library of the package is missing or failed to load."""


class CdsView(C.Structure):
    """``hmxg_cds_view`` (include/hmxg.h)."""

    _fields_ = [
        ("n", C.c_uint64),
        ("num_nodes", C.c_uint32),
        ("height", C.c_uint32),
        ("parent", _u32p),
        ("lchild", _u32p),
        ("rchild", _u32p),
        ("start", _u32p),
        ("end", _u32p),
        ("level", _u32p),
        ("perm", _u32p),
        ("sranks", _u32p),
        ("participating", C.POINTER(C.c_uint8)),
        ("num_near", C.c_uint64),
        ("near_pairs", _u32p),
        ("num_far", C.c_uint64),
        ("far_pairs", _u32p),
        ("num_v", C.c_uint64),
        ("v_order", _u32p),
        ("dptr", _u64p),
        ("bptr", _u64p),
        ("vptr", _u64p),
        ("dgen", _f64p),
        ("bgen", _f64p),
        ("vgen", _f64p),
    ]


class Stats(C.Structure):
    """``hmxg_stats``."""

    _fields_ = [
        ("locked_pairs", C.c_uint64),
        ("seconds", C.c_double),
        ("device_ms", C.c_double),
        ("launches", C.c_uint32),
    ]


class Info(C.Structure):
    """``hmxg_info``."""

    _fields_ = [
        ("n", C.c_uint64),
        ("d_elems", C.c_uint64),
        ("b_elems", C.c_uint64),
        ("v_elems", C.c_uint64),
        ("skel_rows", C.c_uint64),
        ("num_devices", C.c_uint32),
        ("launches_per_eval", C.c_uint32),
        ("flops_per_col", C.c_double),
        ("device_bytes", C.c_uint64),
        ("exec_flops_per_col", C.c_double),
        ("split_parts", C.c_uint32),
        ("part", C.c_uint32),
    ]


# hmxg_allgatherv_fn (include/hmxg.h): user, sendbuf, sendbytes, recvbuf, recvbytes[], displs[], stream
ALLGATHERV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.POINTER(C.c_size_t),
                            C.POINTER(C.c_size_t), C.c_void_p)


class Comm(C.Structure):
    """``hmxg_comm``."""

    _fields_ = [
        ("rank", C.c_uint32),
        ("size", C.c_uint32),
        ("allgatherv", ALLGATHERV_FN),
        ("user", C.c_void_p),
        ("host_buffers", C.c_int32),
        ("reserved", C.c_uint32),
        ("hbm_budget", C.c_uint64),
    ]


class Phase(C.Structure):
    """``hmxg_phase``."""

    _fields_ = [
        ("kind", C.c_uint32),
        ("level", C.c_uint32),
        ("tiles", C.c_uint32),
        ("reserved", C.c_uint32),
        ("flops_per_col", C.c_double),
        ("gen_bytes", C.c_double),
        ("io_bytes_per_col", C.c_double),
        ("last_ms", C.c_double),
    ]


class BuildSpec(C.Structure):
    """``hmxb_spec`` (include/hmxb.h)."""

    _fields_ = [
        ("n", C.c_uint64),
        ("d", C.c_uint32),
        ("points", C.c_int32),
        ("components", C.c_uint32),
        ("levels", C.c_uint32),
        ("seed", C.c_uint64),
        ("kernel", C.c_int32),
        ("h", C.c_double),
        ("leaf", C.c_uint32),
        ("split", C.c_int32),
        ("mode", C.c_int32),
        ("tau", C.c_double),
        ("budget", C.c_double),
        ("max_rank", C.c_uint32),
        ("tol", C.c_double),
        ("sample_rows", C.c_uint32),
        ("knn_k", C.c_uint32),
        ("near_blocksize", C.c_uint32),
        ("far_blocksize", C.c_uint32),
        ("coarsen_p", C.c_uint32),
        ("coarsen_agg", C.c_uint32),
        ("threads", C.c_uint32),
        ("skip_near", C.c_uint32),
    ]


class BuildStats(C.Structure):
    """``hmxb_build_stats``."""

    _fields_ = [
        ("seconds_points", C.c_double),
        ("seconds_tree", C.c_double),
        ("seconds_interactions", C.c_double),
        ("seconds_sampling", C.c_double),
        ("seconds_compress", C.c_double),
        ("seconds_blocks", C.c_double),
        ("seconds_total", C.c_double),
        ("leaves", C.c_uint64),
        ("near_pairs", C.c_uint64),
        ("far_pairs", C.c_uint64),
        ("max_srank", C.c_uint32),
        ("height", C.c_uint32),
    ]


# Exported symbols per library: (name, restype, argtypes). The CPU test suite checks
# that every symbol declared in include/*.h is exported.
HMXG_SYMBOLS = {
    "hmxg_create": (C.c_int, [C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_void_p)]),
    "hmxg_destroy": (C.c_int, [C.c_void_p]),
    "hmxg_create_comm": (C.c_int, [C.c_int, C.POINTER(Comm), C.POINTER(C.c_void_p)]),
    "hmxg_upload": (C.c_int, [C.c_void_p, C.POINTER(CdsView), C.POINTER(C.c_void_p)]),
    "hmxg_free": (C.c_int, [C.c_void_p]),
    "hmxg_validate": (C.c_int, [C.POINTER(CdsView), C.POINTER(Info)]),
    "hmxg_cds_fingerprint": (C.c_int, [C.POINTER(CdsView), C.POINTER(C.c_uint64)]),
    "hmxg_dag_check": (C.c_int, [C.POINTER(CdsView), C.c_size_t, C.c_uint32, C.POINTER(C.c_uint64)]),
    "hmxg_dag_items": (C.c_int, [C.POINTER(CdsView), C.c_size_t, C.c_uint32, C.POINTER(C.c_uint64), C.c_size_t,
                                C.POINTER(C.c_uint64)]),
    "hmxg_info_get": (C.c_int, [C.c_void_p, C.POINTER(Info)]),
    "hmxg_evaluate": (
        C.c_int,
        [C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t, C.c_size_t, C.c_void_p, C.c_size_t,
         C.c_uint, C.c_void_p, C.POINTER(Stats)],
    ),
    "hmxg_upload_generated": (C.c_int, [C.c_void_p, C.POINTER(CdsView), C.c_void_p, C.c_uint32, C.c_int32,
                                        C.c_double, C.POINTER(C.c_uint64), _u32p, C.POINTER(C.c_void_p)]),
    "hmxg_upload_generated_ex": (C.c_int, [C.c_void_p, C.POINTER(CdsView), C.c_void_p, C.c_uint32, C.c_int32,
                                           C.c_double, C.POINTER(C.c_uint64), _u32p, C.c_uint, C.POINTER(C.c_void_p)]),
    "hmxg_upload_split": (C.c_int, [C.c_void_p, C.POINTER(CdsView), C.c_uint32, C.c_uint32, C.POINTER(C.c_void_p)]),
    "hmxg_split_stage": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_size_t, C.c_size_t, C.c_size_t, C.c_void_p,
                                   C.c_size_t, C.c_void_p]),
    "hmxg_split_exchange_buffer": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]),
    "hmxg_split_exchange": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]),
    "hmxg_phase_count": (C.c_int, [C.c_void_p]),
    "hmxg_phase_get": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(Phase)]),
    "hmxg_cds_file_open": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "hmxg_cds_file_view": (C.c_int, [C.c_void_p, C.POINTER(CdsView)]),
    "hmxg_cds_file_header": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint32), C.POINTER(C.c_double),
                                       C.POINTER(C.c_uint32)]),
    "hmxg_cds_file_close": (None, [C.c_void_p]),
    "hmxg_cds_file_error": (C.c_char_p, []),
    "hmxg_points_upload": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_int32, C.c_double,
                                     C.POINTER(C.c_void_p)]),
    "hmxg_points_free": (C.c_int, [C.c_void_p]),
    "hmxg_kernel_rows": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_size_t, C.c_size_t,
                                   C.c_size_t, C.c_void_p, C.c_size_t, C.c_uint, C.c_void_p, C.POINTER(Stats)]),
    "hmxg_sample_rows": (C.c_uint64, [C.c_uint64, C.c_uint64, C.c_void_p]),
    "hmxg_relative_error": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t, C.c_size_t,
                                      C.c_size_t, C.c_int, C.c_uint64, C.c_uint, C.POINTER(C.c_double)]),
    "hmxg_compress": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_int32, C.c_double, C.c_uint32,
                                _u32p, _u32p, _u32p, _u32p, _u32p, _u32p, C.POINTER(C.c_uint8),
                                C.POINTER(C.c_uint64), _u32p, C.c_double, C.c_uint32, C.POINTER(C.c_void_p)]),
    "hmxg_compressed_get": (C.c_int, [C.c_void_p, C.POINTER(_u32p), C.POINTER(C.POINTER(C.c_uint64)),
                                      C.POINTER(_u32p), C.POINTER(C.POINTER(C.c_uint64)),
                                      C.POINTER(C.POINTER(C.c_uint64)), C.POINTER(_f64p)]),
    "hmxg_compressed_free": (None, [C.c_void_p]),
    "hmxg_last_error": (C.c_char_p, []),
    "hmxg_version": (C.c_char_p, []),
}
HMXB_SYMBOLS = {
    "hmxb_spec_default": (None, [C.POINTER(BuildSpec)]),
    "hmxb_build": (C.c_int, [C.POINTER(BuildSpec), C.POINTER(C.c_void_p)]),
    "hmxb_view": (C.c_int, [C.c_void_p, C.POINTER(CdsView)]),
    "hmxb_points": (C.c_int, [C.c_void_p, C.POINTER(_f64p), C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)]),
    "hmxb_stats": (C.c_int, [C.c_void_p, C.POINTER(BuildStats)]),
    "hmxb_dense_rows": (
        C.c_int,
        [C.c_void_p, _u32p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_uint64],
    ),
    "hmxb_free": (None, [C.c_void_p]),
    "hmxb_random_w": (None, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p]),
    "hmxb_last_error": (C.c_char_p, []),
}

_lock = threading.Lock()
_libs: dict[str, C.CDLL] = {}


def _load(path: str, symbols: dict) -> C.CDLL:
    with _lock:
        if path in _libs:
            return _libs[path]
        if not os.path.exists(path):
            raise NativeLibraryError(
                f"{os.path.basename(path)} is not built ({path}); run "
                "`python -c 'import __graft_entry__ as g; g.build()'` first")
        try:
            lib = C.CDLL(path, mode=C.RTLD_GLOBAL)
        except OSError as e:  # pragma: no cover - depends on the box
            raise NativeLibraryError(f"cannot load {path}: {e}") from e
        for name, (res, args) in symbols.items():
            fn = getattr(lib, name, None)  # an older A/B build (HMXG_LIBRARY) may lack newer entry points
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        _libs[path] = lib
        return lib


def hmxg() -> C.CDLL:
    """The evaluator library (raises if missing: the CUDA path has no fallback)."""
    return _load(HMXG_PATH, HMXG_SYMBOLS)


def hmxb() -> C.CDLL:
    """The host instance builder library."""
    return _load(HMXB_PATH, HMXB_SYMBOLS)


def last_error(lib: C.CDLL, prefix: str) -> str:
    msg = getattr(lib, prefix + "_last_error")()
    return msg.decode() if msg else "unknown error"
