"""ctypes binding of include/fvsr_b200.h (the C-ABI of libfvsr_b200.so).

The library is built in-tree (``python -m paper_2510_12747_b200.build``).  There is no
fallback: if the .so is missing or the device is not an sm_100 B200, every compute entry
point raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from . import build as _build

LIB_PATH = _build.LIB

FVSR_OK = 0
FVSR_E_SHAPE = 1
FVSR_E_CONFIG = 2
FVSR_E_DEGENERATE = 3
FVSR_E_EMPTY_BLOCK = 4
FVSR_E_INVARIANT = 5
FVSR_E_CUDA = 6
FVSR_E_NOMEM = 8

MASK_ALL, MASK_LOCALITY, MASK_BITMASK = 0, 1, 2
LOCALITY_PRESERVED, LOCALITY_TRUNCATED = 0, 1
FLAG_SYNC_CHECK = 1
FLAG_NO_TMA = 2
OUT_TOKEN_MAJOR, OUT_TILE_MAJOR = 0, 1
TIME_APPEND, TIME_MASK_BUILDER, TIME_ATTENTION, TIME_FRONT, TIME_PACK, TIME_SELECT = 0, 1, 2, 3, 4, 5


class Error(RuntimeError):
    """Base of the reference's error taxonomy (P/include/vsr/common.hpp:10-13)."""


class ShapeError(Error):
    pass


class ConfigError(Error):
    pass


class DegenerateRowError(Error):
    pass


class EmptyBlockError(Error):
    pass


class InvariantError(Error):
    pass


class CudaError(Error):
    pass


_EXC = {FVSR_E_SHAPE: ShapeError, FVSR_E_CONFIG: ConfigError, FVSR_E_DEGENERATE: DegenerateRowError,
        FVSR_E_EMPTY_BLOCK: EmptyBlockError, FVSR_E_INVARIANT: InvariantError, FVSR_E_CUDA: CudaError,
        FVSR_E_NOMEM: CudaError}


class Grid(C.Structure):
    _fields_ = [("frame_ids", C.POINTER(C.c_int32)), ("n_frames", C.c_int32), ("rows", C.c_int32),
                ("cols", C.c_int32)]


class MaskDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("mode", C.c_int32), ("extent_h", C.c_int32), ("extent_w", C.c_int32),
                ("bits", C.c_void_p), ("words_per_row", C.c_int64)]


P = C.c_void_p
I32, I64, F32 = C.c_int32, C.c_int64, C.c_float
GP = C.POINTER(Grid)
MP = C.POINTER(MaskDesc)


class Layout(C.Structure):
    """fvsr_layout: element strides of head h / token t (include/fvsr_b200.h); {0, 0} = [heads][L][d]."""
    _fields_ = [("head_stride", C.c_int64), ("token_stride", C.c_int64)]


LAYOUT = Layout

# name -> (restype, argtypes); must list every symbol include/fvsr_b200.h declares
SIGNATURES = {
    "fvsr_abi_version": (I32, []),
    "fvsr_last_error": (C.c_char_p, []),
    "fvsr_ctx_create": (I32, [C.POINTER(P)]),
    "fvsr_ctx_destroy": (None, [P]),
    "fvsr_ctx_set_flags": (I32, [P, I32]),
    "fvsr_check_errors": (I32, [P, P]),
    "fvsr_ctx_launch_count": (I64, [P]),
    "fvsr_ctx_timing_enable": (I32, [P, I32]),
    "fvsr_ctx_timing_read": (I32, [P, I32, C.POINTER(C.c_double), C.POINTER(I64), I32]),
    "fvsr_ctx_read_pairs": (I32, [P, C.POINTER(C.c_uint64)]),
    "fvsr_block_counts": (I32, [GP, GP, C.POINTER(I32), C.POINTER(I32)]),
    "fvsr_plan_sparse": (I32, [P, P, P, I32, I32, GP, GP, MP, I64, I32, P, P, P, P, P, P]),
    "fvsr_sparse_attention_exec": (I32, [P, P, P, P, I32, I32, GP, GP, MP, I32, P, P, F32, I64, I64, P, P]),
    "fvsr_sparsity_report": (I32, [P, I32, GP, GP, MP, I32, P, P, P, P, P, P, P]),
    "fvsr_ring_create": (I32, [P, I32, I32, I32, I32, I32, I32, C.POINTER(P)]),
    "fvsr_ring_destroy": (None, [P]),
    "fvsr_ring_append": (I32, [P, P, I32, I32, P, P, P]),
    "fvsr_ring_set_rope": (I32, [P, C.c_double, C.POINTER(I32)]),
    "fvsr_ring_evict_sliding": (I32, [P, I32]),
    "fvsr_ring_evict_keep": (I32, [P, I32, I32]),
    "fvsr_ring_frame_ids": (I32, [P, I32, C.POINTER(I32), I32, C.POINTER(I32)]),
    "fvsr_ring_attention": (I32, [P, P, I32, P, C.POINTER(I32), I32, MP, I64, F32, I64, I64, P, I32, I32, P, P,
                                  P]),
    "fvsr_build_segment_mask": (I32, [P, C.POINTER(I32), I64, P, P]),
    "fvsr_build_causal_mask": (I32, [P, C.POINTER(I32), I64, I32, P, P]),
    "fvsr_frame_attention_mass": (I32, [P, I32, GP, GP, MP, P, P, P]),
    "fvsr_ring_frame_mass": (I32, [P, P, I32, C.POINTER(I32), I32, MP, P, P]),
    "fvsr_ring_evict": (I32, [P, I32, I32, P]),
    "fvsr_build_flags": (C.c_char_p, []),
    "fvsr_ring_frame_ids_head": (I32, [P, I32, I32, C.POINTER(I32), I32, C.POINTER(I32)]),
    "fvsr_rms_norm": (I32, [P, P, P, I64, I32, P, P]),
    "fvsr_ring_step_layout": (I32, [P, P, I32, I32, P, P, LAYOUT, P, LAYOUT, C.POINTER(I32), I32, MP, I64, F32, P,
                                    LAYOUT, P]),
    "fvsr_untile": (I32, [P, P, I64, I32, I32, I32, I32, I32, P, P]),
    "fvsr_plan_sparse_f32": (I32, [P, P, P, I32, I32, GP, GP, MP, I64, I32, P, P, P, P, P, P]),
    "fvsr_ring_step": (I32, [P, P, I32, I32, P, P, P, C.POINTER(I32), I32, MP, I64, F32, I64, I64, P, I32, I32, P,
                             P, P]),
    "fvsr_ctx_read_tiles": (I32, [P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "fvsr_ring_step_host": (I32, [P, P, I32, I32, P, P, P, MP, I64, F32, P, P]),
}

_lib = None
_lock = threading.Lock()


def load(build_if_missing: bool = True):
    """Load libfvsr_b200.so (rebuilding it in-tree if missing or older than its sources) and
    bind every C-ABI symbol.  FVSR_LIB=<path> loads an experiment variant instead (see
    build.build_variant); a library built with experiment macros is refused otherwise."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = os.environ.get("FVSR_LIB") or LIB_PATH
        if path == LIB_PATH and _build.stale():
            if not os.path.exists(LIB_PATH) and not build_if_missing:
                raise ImportError(f"{LIB_PATH} is missing; run `python -m paper_2510_12747_b200.build`")
            if os.path.exists(os.path.join(_build.HERE, "csrc")) and os.access(_build.HERE, os.W_OK):
                try:
                    _build.build()
                except Exception:
                    if not os.path.exists(LIB_PATH):
                        raise
        lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.fvsr_abi_version() != 1:
            raise ImportError("libfvsr_b200.so ABI version mismatch")
        flags = lib.fvsr_build_flags().decode()
        if flags and not os.environ.get("FVSR_LIB"):
            raise ImportError(f"{path} is an experiment build ({flags}); rebuild with "
                              "`python -m paper_2510_12747_b200.build --force`")
        _lib = lib
        return lib


def check(status: int) -> None:
    if status == FVSR_OK:
        return
    msg = load().fvsr_last_error()
    msg = msg.decode() if msg else ""
    raise _EXC.get(status, Error)(msg)


def make_grid(frame_ids, rows: int, cols: int):
    """Return (Grid, keepalive) for a host frame-id list (== vsr::TokenGrid)."""
    ids = (C.c_int32 * max(1, len(frame_ids)))(*[int(f) for f in frame_ids])
    return Grid(C.cast(ids, C.POINTER(C.c_int32)), len(frame_ids), int(rows), int(cols)), ids
