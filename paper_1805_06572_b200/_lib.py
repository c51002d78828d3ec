"""ctypes binding of libfastfca_b200.so (the C ABI in include/fastfca_b200.h).

The library is built in-tree (``python -m paper_1805_06572_b200.build``) and
loaded from ``paper_1805_06572_b200/lib/``. There is no fallback: if the
library is missing, loading raises :class:`BackendUnavailableError`.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import BackendUnavailableError

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libfastfca_b200.so"

FFCA_OK = 0
FFCA_ERR_SINGULAR_MATRIX = 1
FFCA_ERR_SINGULAR_MIXTURE = 2
FFCA_ERR_DEFINITENESS = 3
FFCA_ERR_NON_HERMITIAN = 4
FFCA_ERR_SINGULAR_BASIS = 5
FFCA_ERR_NOT_PD = 6
FFCA_ERR_NO_CONVERGENCE = 7
FFCA_ERR_INVALID = 10
FFCA_ERR_CUDA = 11

FFCA_C128 = 0
FFCA_C64 = 1

FLAG_LIKELIHOOD = 1
FLAG_HISTORY = 2
FLAG_IMAGES = 4
FLAG_GRAPH = 8
FLAG_PERSIST = 16
FLAG_NO_PERSIST = 32

c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_vp = ctypes.c_void_p
c_sz = ctypes.c_size_t


class StatusDev(ctypes.Structure):
    _fields_ = [("first", ctypes.c_ulonglong), ("value", ctypes.c_double)]


class Status(ctypes.Structure):
    _fields_ = [("code", c_int), ("iteration", c_int), ("index", ctypes.c_longlong),
                ("value", ctypes.c_double)]


class RunArgs(ctypes.Structure):
    _fields_ = [
        ("M", c_i64), ("N", c_i64), ("F", c_i64),
        ("I", c_int), ("dtype", c_int), ("iterations", c_int), ("flags", ctypes.c_uint),
        ("y", c_vp), ("v", c_vp), ("S0", c_vp), ("v_floor", c_vp), ("images", c_vp),
        ("S_out", c_vp), ("loglik", c_vp), ("S_hist", c_vp), ("v_hist", c_vp),
        ("workspace", c_vp), ("workspace_bytes", c_sz), ("iter_events", c_vp),
        ("chunk_frames", c_i64), ("kernel_events", c_vp), ("v_in", c_vp),
        ("bin_parts", c_int),
    ]


# (name, restype, argtypes) for every symbol the header declares
SIGNATURES = [
    ("ffca_version", ctypes.c_char_p, []),
    ("ffca_device_arch", c_int, []),
    ("ffca_plan_chunks", c_int,
     [c_i64, c_i64, c_int, c_int, c_int, ctypes.POINTER(c_i64), ctypes.POINTER(c_int)]),
    ("ffca_plan_parts", c_int, [c_i64, c_i64, c_int, c_int, c_int]),
    ("ffca_plan_grid", c_int,
     [c_i64, c_i64, c_int, c_int, c_int, c_i64, ctypes.POINTER(c_i64), ctypes.POINTER(c_i64)]),
    ("ffca_fastfca_workspace_size", c_sz,
     [c_i64, c_i64, c_i64, c_int, c_int, ctypes.c_uint, c_i64]),
    ("ffca_fastfca_run", c_int, [ctypes.POINTER(RunArgs), c_vp]),
    ("ffca_fca_workspace_size", c_sz, [c_i64, c_i64, c_i64, c_int, c_int, ctypes.c_uint, c_i64]),
    ("ffca_fca_run", c_int, [ctypes.POINTER(RunArgs), c_vp]),
    ("ffca_graph_cache_clear", c_int, []),
    ("ffca_run_status", c_int, [c_vp, c_vp, ctypes.POINTER(Status)]),
    ("ffca_status_reset", c_int, [c_vp, c_vp]),
    ("ffca_status_read", c_int, [c_vp, c_vp, ctypes.POINTER(Status)]),
    ("ffca_status_decode", c_int, [c_vp, ctypes.POINTER(Status)]),
    ("ffca_fast_transform", c_int, [c_vp, c_vp, c_vp, c_i64, c_i64, c_int, c_vp]),
    ("ffca_fast_e_step", c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_int, c_vp]),
    ("ffca_fast_v_update", c_int, [c_vp, c_vp, c_vp, c_i64, c_i64, c_int, c_vp]),
    ("ffca_S_update", c_int, [c_vp, c_vp, c_vp, c_i64, c_i64, c_int, c_vp]),
    ("ffca_fast_log_likelihood", c_int,
     [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_int, c_vp]),
    ("ffca_fast_iteration", c_int,
     [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_int, c_vp, c_vp]),
    ("ffca_fca_e_step", c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_int, c_vp, c_vp]),
    ("ffca_fca_v_update", c_int, [c_vp, c_vp, c_vp, c_i64, c_i64, c_int, c_vp, c_vp]),
    ("ffca_fca_log_likelihood", c_int,
     [c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_int, c_vp, c_vp]),
    ("ffca_fca_iteration", c_int,
     [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_int, c_vp, c_vp]),
    ("ffca_gevd_hpd", c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_int, c_int, c_vp, c_vp]),
    ("ffca_propagate_pencil", c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_int, c_vp, c_vp]),
    ("ffca_cholesky_inverse", c_int, [c_vp, c_vp, c_i64, c_int, c_vp, c_vp]),
    ("ffca_solve", c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_int, c_i64, c_vp, c_vp]),
    ("ffca_regularize_covariances", c_int, [c_vp, c_vp, c_i64, c_int, c_vp]),
    ("ffca_regularize_transformed", c_int, [c_vp, c_vp, c_vp, c_i64, c_int, c_vp]),
    ("ffca_back_transform_images", c_int,
     [c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_int, c_vp, c_vp]),
    ("ffca_back_transform_covariances", c_int,
     [c_vp, c_vp, c_vp, c_i64, c_i64, c_int, c_vp, c_vp]),
    ("ffca_logdet2", c_int, [c_vp, c_vp, c_i64, c_int, c_vp]),
    ("ffca_init_powers", c_int, [c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_int, c_int, c_vp]),
    ("ffca_init_masks_workspace_size", c_sz, [c_i64, c_i64, c_i64, c_int]),
    ("ffca_init_masks", c_int,
     [c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_int, c_vp, c_sz, c_vp]),
    ("ffca_stft_frames", c_i64, [c_i64, c_int]),
    ("ffca_stft_analyze", c_int, [c_vp, c_vp, c_i64, c_int, c_i64, c_int, c_vp]),
    ("ffca_stft_synthesize", c_int, [c_vp, c_vp, c_i64, c_int, c_i64, c_int, c_i64, c_vp]),
    ("ffca_sdr_workspace_size", c_sz, [c_i64, c_i64, c_int]),
    ("ffca_sdr", c_int, [c_vp, c_vp, c_i64, c_i64, c_int, c_vp, c_vp, c_vp, c_vp]),
]

_lib = None


def load(path: os.PathLike | None = None):
    """Load (once) and return the ctypes library handle, with signatures set."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else Path(os.environ.get("FFCA_LIBRARY", LIB_PATH))
    if not p.exists():
        raise BackendUnavailableError(
            f"{p} is missing: build it with `python -m paper_1805_06572_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(str(p))
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib
