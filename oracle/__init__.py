"""TEST INFRASTRUCTURE ONLY — CPU oracles for the FlashVSR block-sparse hot path.

Two checkers, both host-only, both used *only* by ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs (never by the product package ``paper_2510_12747_b200``):

* ``Port`` — ``oracle/fvsr_port.c``, a plain-C restatement of the reference
  algorithm (each function cites /root/reference/proj file:line).  Always
  buildable (``make -C oracle port``).
* ``Ref`` — ``oracle/_ref/libvsr_ref.so``, the UNMODIFIED reference sources
  (P/src/{tensor,mask,partition,attention,sparse}.cpp) compiled read-only from
  /root/reference by ``oracle/Makefile`` plus an extern-C shim
  (``oracle/ref_shim.cpp``).  Built here (the reference tree exists only in the
  build container); the .so travels to the GPU box with the repo snapshot.

Parity is pinned: ``tests/test_oracle.py`` checks Port == Ref bit-for-bit on
seeded cases and both against the committed fixtures in ``tests/golden/``.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libfvsr_port.so")
REF_SO = os.path.join(HERE, "_ref", "libvsr_ref.so")
REF_TREE = "/root/reference/proj"

ERRORS = {1: "ShapeError", 2: "ConfigError", 3: "DegenerateRowError",
          4: "EmptyBlockError", 5: "InvariantError", 8: "NoMemory", 9: "Error"}


class OracleError(RuntimeError):
    """Reference exception mapped through the C shim; ``kind`` names the type."""

    def __init__(self, code: int, msg: str = ""):
        self.code = code
        self.kind = ERRORS.get(code, f"code{code}")
        super().__init__(f"{self.kind}: {msg}")


def build(ref: Optional[bool] = None) -> None:
    """Build the port (always) and the reference shim (when the tree exists)."""
    subprocess.run(["make", "-s", "-C", HERE, "port"], check=True)
    if ref is None:
        ref = os.path.isdir(REF_TREE)
    if ref:
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


# ----------------------------------------------------------------------------
# Case description shared by both oracles
# ----------------------------------------------------------------------------

@dataclass
class Mask:
    kind: int = 0            # 0 all-allowed, 1 locality, 2 bitmask
    mode: int = 1            # 0 boundary_preserved, 1 boundary_truncated
    extent_h: int = 1
    extent_w: int = 1
    bits: Optional[np.ndarray] = None   # uint64 [Lq][words_per_row]

    @staticmethod
    def all() -> "Mask":
        return Mask(0)

    @staticmethod
    def locality(extent_h: int, extent_w: int, truncated: bool = True) -> "Mask":
        return Mask(1, 1 if truncated else 0, extent_h, extent_w)

    @staticmethod
    def bitmask(bits: np.ndarray) -> "Mask":
        return Mask(2, 0, 1, 1, np.ascontiguousarray(bits, dtype=np.uint64))


@dataclass
class Plan:
    sel: np.ndarray          # int32 [bnq][cap], ascending, -1 padded
    count: np.ndarray        # int32 [bnq]
    diag: np.ndarray         # int32 [bnq]
    coarse: np.ndarray       # float32 [bnq][bnk]
    allowed: np.ndarray      # uint8 [bnq][bnk]

    @property
    def bnq(self) -> int:
        return self.sel.shape[0]

    def lists(self):
        return [list(map(int, self.sel[i, : self.count[i]])) for i in range(self.bnq)]


def block_count(frame_ids: Sequence[int], rows: int, cols: int) -> int:
    """Number of (2,8,8) blocks partition_blocks produces (P/src/partition.cpp:38-62)."""
    keys = {(f // 2, h // 8, w // 8) for f in frame_ids for h in range(0, rows, 8) for w in range(0, cols, 8)}
    return len(keys)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


# ----------------------------------------------------------------------------
# Port (plain-C restatement)
# ----------------------------------------------------------------------------

class _FpGrid(C.Structure):
    _fields_ = [("frame_ids", C.POINTER(C.c_int)), ("n_frames", C.c_int),
                ("rows", C.c_int), ("cols", C.c_int)]


class _FpMask(C.Structure):
    _fields_ = [("kind", C.c_int), ("mode", C.c_int), ("extent_h", C.c_int),
                ("extent_w", C.c_int), ("bits", C.POINTER(C.c_uint64)),
                ("words_per_row", C.c_long)]


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(C.POINTER(t))


class Port:
    """ctypes facade over oracle/_build/libfvsr_port.so."""

    _lib = None

    def __init__(self):
        if Port._lib is None:
            if not os.path.exists(PORT_SO):
                build(ref=False)
            lib = C.CDLL(PORT_SO)
            lib.fp_gaussian.argtypes = [C.c_uint64, C.POINTER(C.c_float), C.c_long]
            lib.fp_gaussian.restype = None
            Port._lib = lib
        self.lib = Port._lib
        self._keep = []

    # -- helpers ------------------------------------------------------------
    def _grid(self, frame_ids, rows, cols):
        ids = _i32(frame_ids)
        self._keep.append(ids)
        return _FpGrid(_ptr(ids, C.c_int), len(ids), rows, cols)

    def _mask(self, m: Mask, lk: int):
        if m.kind == 2:
            bits = np.ascontiguousarray(m.bits, dtype=np.uint64)
            self._keep.append(bits)
            return _FpMask(2, m.mode, m.extent_h, m.extent_w, _ptr(bits, C.c_uint64), (lk + 63) // 64)
        return _FpMask(m.kind, m.mode, m.extent_h, m.extent_w, None, (lk + 63) // 64)

    # -- API ----------------------------------------------------------------
    def gaussian(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.float32)
        self.lib.fp_gaussian(seed, _ptr(out, C.c_float), n)
        return out

    def partition(self, frame_ids, rows, cols):
        L = len(frame_ids) * rows * cols
        assign = np.empty(L, np.int32)
        keys = np.empty((L, 3), np.int32)
        nb = C.c_int()
        g = self._grid(frame_ids, rows, cols)
        st = self.lib.fp_partition(C.byref(g), _ptr(assign, C.c_int), _ptr(keys, C.c_int), C.byref(nb))
        if st:
            raise OracleError(st)
        return assign, keys[: nb.value].copy()

    def plan(self, q, k, qf, kf, rows, cols, mask: Mask, topk: int) -> Plan:
        q, k = _f32(q), _f32(k)
        d = q.shape[1]
        bnq, bnk = block_count(qf, rows, cols), block_count(kf, rows, cols)
        cap = max(1, min(int(topk), bnk))
        sel = np.full((bnq, cap), -1, np.int32)
        cnt = np.zeros(bnq, np.int32)
        diag = np.zeros(bnq, np.int32)
        coarse = np.zeros((bnq, bnk), np.float32)
        allowed = np.zeros((bnq, bnk), np.uint8)
        gq, gk = self._grid(qf, rows, cols), self._grid(kf, rows, cols)
        mk = self._mask(mask, k.shape[0])
        st = self.lib.fp_plan(_ptr(q, C.c_float), _ptr(k, C.c_float), C.c_int(d), C.byref(gq),
                              C.byref(gk), C.byref(mk), C.c_long(int(topk)), C.c_int(cap),
                              _ptr(sel, C.c_int), _ptr(cnt, C.c_int), _ptr(diag, C.c_int),
                              _ptr(coarse, C.c_float), _ptr(allowed, C.c_uint8))
        self._keep.clear()
        if st:
            raise OracleError(st)
        return Plan(sel, cnt, diag, coarse, allowed)

    def exec(self, q, k, v, qf, kf, rows, cols, mask: Mask, plan: Plan, scale: float,
             row_begin: int = 0, row_end: int = -1) -> np.ndarray:
        q, k, v = _f32(q), _f32(k), _f32(v)
        d = q.shape[1]
        out = np.zeros_like(q)
        sel, cnt = _i32(plan.sel), _i32(plan.count)
        gq, gk = self._grid(qf, rows, cols), self._grid(kf, rows, cols)
        mk = self._mask(mask, k.shape[0])
        st = self.lib.fp_exec(_ptr(q, C.c_float), _ptr(k, C.c_float), _ptr(v, C.c_float), C.c_int(d),
                              C.byref(gq), C.byref(gk), C.byref(mk), C.c_int(sel.shape[1]),
                              _ptr(sel, C.c_int), _ptr(cnt, C.c_int), C.c_float(scale),
                              C.c_long(row_begin), C.c_long(row_end), _ptr(out, C.c_float))
        self._keep.clear()
        if st:
            raise OracleError(st)
        return out

    def report(self, qf, kf, rows, cols, mask: Mask, plan: Plan, lk: int):
        sel, cnt = _i32(plan.sel), _i32(plan.count)
        gq, gk = self._grid(qf, rows, cols), self._grid(kf, rows, cols)
        mk = self._mask(mask, lk)
        ex, dense, ns, na = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        st = self.lib.fp_report(C.byref(gq), C.byref(gk), C.byref(mk), C.c_int(sel.shape[1]),
                                _ptr(sel, C.c_int), _ptr(cnt, C.c_int), C.byref(ex), C.byref(dense),
                                C.byref(ns), C.byref(na))
        self._keep.clear()
        if st:
            raise OracleError(st)
        return {"executed_pairs": ex.value, "dense_pairs": dense.value,
                "selected_blocks": ns.value, "allowed_blocks": na.value,
                "density": ns.value / na.value if na.value else 0.0}


# ----------------------------------------------------------------------------
# Ref (compiled reference + shim)
# ----------------------------------------------------------------------------

class Ref:
    """ctypes facade over oracle/_ref/libvsr_ref.so (the unmodified reference)."""

    _lib = None

    def __init__(self):
        if Ref._lib is None:
            if not os.path.exists(REF_SO):
                if not os.path.isdir(REF_TREE):
                    raise FileNotFoundError("oracle/_ref not built and /root/reference absent")
                build(ref=True)
            lib = C.CDLL(REF_SO)
            lib.vsrref_gaussian.argtypes = [C.c_uint64, C.POINTER(C.c_float), C.c_size_t]
            lib.vsrref_gaussian.restype = None
            lib.vsrref_case_new.restype = C.c_void_p
            lib.vsrref_case_free.argtypes = [C.c_void_p]
            lib.vsrref_case_dims.argtypes = [C.c_void_p] + [C.POINTER(C.c_int)] * 5
            lib.vsrref_mask_bits.argtypes = [C.c_void_p, C.POINTER(C.c_uint64)]
            lib.vsrref_plan.argtypes = [C.c_void_p, C.c_long, C.c_char_p, C.c_int]
            lib.vsrref_plan_get.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                            C.POINTER(C.c_int), C.POINTER(C.c_float), C.POINTER(C.c_uint8)]
            lib.vsrref_plan_set_selection.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
            lib.vsrref_exec.argtypes = [C.c_void_p, C.c_float, C.c_long, C.c_long, C.c_uint,
                                        C.POINTER(C.c_float), C.c_char_p, C.c_int]
            lib.vsrref_report.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_uint64),
                                          C.POINTER(C.c_uint64), C.c_char_p, C.c_int]
            lib.vsrref_dense.argtypes = [C.c_void_p, C.c_float, C.POINTER(C.c_float), C.c_char_p, C.c_int]
            lib.vsrref_dense_stream.argtypes = [C.c_void_p, C.c_float, C.c_long, C.POINTER(C.c_float), C.c_char_p,
                                                C.c_int]
            lib.vsrref_apply_rope.argtypes = [C.POINTER(C.c_int), C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                              C.POINTER(C.c_int), C.POINTER(C.c_float), C.c_char_p, C.c_int]
            lib.vsrref_segment_mask.argtypes = [C.POINTER(C.c_int), C.c_long, C.POINTER(C.c_uint64), C.c_char_p,
                                                C.c_int]
            lib.vsrref_causal_mask.argtypes = [C.POINTER(C.c_int), C.c_long, C.c_int, C.POINTER(C.c_uint64),
                                               C.c_char_p, C.c_int]
            lib.vsrref_frame_mass.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_char_p, C.c_int]
            lib.vsrref_kv_evict.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int),
                                            C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                            C.c_char_p, C.c_int]
            lib.vsrref_head_attention.argtypes = [C.c_void_p, C.c_long, C.c_float, C.c_uint, C.c_int,
                                                  C.c_int, C.c_int, C.c_int, C.POINTER(C.c_float),
                                                  C.c_char_p, C.c_int]
            Ref._lib = lib
        self.lib = Ref._lib

    def gaussian(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.float32)
        self.lib.vsrref_gaussian(seed, _ptr(out, C.c_float), n)
        return out

    class Case:
        def __init__(self, lib, q, k, v, qf, kf, rows, cols, mask: Mask):
            self.lib = lib
            self.q, self.k, self.v = _f32(q), _f32(k), _f32(v)
            self.qf, self.kf = _i32(qf), _i32(kf)
            self.rows, self.cols = rows, cols
            self.mask = mask
            st = C.c_int()
            err = C.create_string_buffer(512)
            bits = None
            if mask.kind == 2:
                bits = np.ascontiguousarray(mask.bits, dtype=np.uint64)
            self._bits = bits
            self.h = lib.vsrref_case_new(
                _ptr(self.qf, C.c_int), len(self.qf), _ptr(self.kf, C.c_int), len(self.kf), rows, cols,
                self.q.shape[1], _ptr(self.q, C.c_float), _ptr(self.k, C.c_float), _ptr(self.v, C.c_float),
                mask.kind, mask.mode, mask.extent_h, mask.extent_w,
                _ptr(bits, C.c_uint64) if bits is not None else None, C.byref(st), err, 512)
            if st.value:
                raise OracleError(st.value, err.value.decode())
            dims = [C.c_int() for _ in range(5)]
            lib.vsrref_case_dims(self.h, *[C.byref(x) for x in dims])
            self.lq, self.lk, self.bnq, self.bnk, self.wpr = [x.value for x in dims]
            self.cap = None

        def __del__(self):
            if getattr(self, "h", None):
                self.lib.vsrref_case_free(self.h)
                self.h = None

        def mask_bits(self) -> np.ndarray:
            out = np.zeros((self.lq, self.wpr), np.uint64)
            self.lib.vsrref_mask_bits(self.h, _ptr(out, C.c_uint64))
            return out

        def plan(self, topk: int) -> Plan:
            err = C.create_string_buffer(512)
            st = self.lib.vsrref_plan(self.h, int(topk), err, 512)
            if st:
                raise OracleError(st, err.value.decode())
            cap = max(1, min(int(topk), self.bnk))
            self.cap = cap
            sel = np.full((self.bnq, cap), -1, np.int32)
            cnt = np.zeros(self.bnq, np.int32)
            diag = np.zeros(self.bnq, np.int32)
            coarse = np.zeros((self.bnq, self.bnk), np.float32)
            allowed = np.zeros((self.bnq, self.bnk), np.uint8)
            st = self.lib.vsrref_plan_get(self.h, cap, _ptr(sel, C.c_int), _ptr(cnt, C.c_int),
                                          _ptr(diag, C.c_int), _ptr(coarse, C.c_float),
                                          _ptr(allowed, C.c_uint8))
            if st:
                raise OracleError(st)
            return Plan(sel, cnt, diag, coarse, allowed)

        def set_selection(self, plan: Plan) -> None:
            sel, cnt = _i32(plan.sel), _i32(plan.count)
            st = self.lib.vsrref_plan_set_selection(self.h, sel.shape[1], _ptr(sel, C.c_int), _ptr(cnt, C.c_int))
            if st:
                raise OracleError(st)

        def exec(self, scale: float, row_begin: int = 0, row_end: int = -1, threads: int = 1) -> np.ndarray:
            out = np.zeros((self.lq, self.q.shape[1]), np.float32)
            err = C.create_string_buffer(512)
            st = self.lib.vsrref_exec(self.h, scale, row_begin, row_end, threads, _ptr(out, C.c_float), err, 512)
            if st:
                raise OracleError(st, err.value.decode())
            return out

        def report(self):
            dens, ex, dn = C.c_double(), C.c_uint64(), C.c_uint64()
            err = C.create_string_buffer(512)
            st = self.lib.vsrref_report(self.h, C.byref(dens), C.byref(ex), C.byref(dn), err, 512)
            if st:
                raise OracleError(st, err.value.decode())
            return {"density": dens.value, "executed_flops": ex.value, "dense_flops": dn.value}

        def frame_mass(self) -> np.ndarray:
            """vsr::frame_attention_mass(plan, grid_k) (P/src/kv_cache.cpp:170-206)."""
            out = np.zeros(len(self.kf), np.float64)
            err = C.create_string_buffer(512)
            st = self.lib.vsrref_frame_mass(self.h, _ptr(out, C.c_double), err, 512)
            if st:
                raise OracleError(st, err.value.decode())
            return out

        def dense_stream(self, scale: float, rows: int) -> np.ndarray:
            """dense_attention_stream (P/src/attention.cpp:58-99) on the first `rows` query rows."""
            rows = min(int(rows), self.lq)
            out = np.zeros((rows, self.q.shape[1]), np.float32)
            err = C.create_string_buffer(512)
            st = self.lib.vsrref_dense_stream(self.h, C.c_float(scale), C.c_long(rows), _ptr(out, C.c_float), err, 512)
            if st:
                raise OracleError(st, err.value.decode())
            return out

        def dense(self, scale: float) -> np.ndarray:
            out = np.zeros((self.lq, self.q.shape[1]), np.float32)
            err = C.create_string_buffer(512)
            st = self.lib.vsrref_dense(self.h, scale, _ptr(out, C.c_float), err, 512)
            if st:
                raise OracleError(st, err.value.decode())
            return out

        def head_attention(self, topk: int, scale: float, threads: int, out: Optional[np.ndarray] = None):
            err = C.create_string_buffer(512)
            m = self.mask
            st = self.lib.vsrref_head_attention(self.h, int(topk), scale, threads, m.kind if m.kind == 1 else 0,
                                                m.mode, m.extent_h, m.extent_w,
                                                _ptr(out, C.c_float) if out is not None else None, err, 512)
            if st:
                raise OracleError(st, err.value.decode())

    def apply_rope(self, x, frame_ids, rows: int, cols: int, theta0: float = 10000.0, axis_split=None):
        """vsr::apply_rope over TokenGrid(frame_ids, rows, cols).positions() (P/src/rope.cpp:30-62)."""
        x = np.array(x, dtype=np.float32, copy=True, order="C")
        fids = _i32(frame_ids)
        sp = None if axis_split is None else _i32(axis_split)
        err = C.create_string_buffer(512)
        st = self.lib.vsrref_apply_rope(_ptr(fids, C.c_int), len(fids), rows, cols, x.shape[1], float(theta0),
                                        _ptr(sp, C.c_int) if sp is not None else None, _ptr(x, C.c_float), err, 512)
        if st:
            raise OracleError(st, err.value.decode())
        return x

    def segment_mask(self, seg) -> np.ndarray:
        """vsr::build_segment_mask (P/src/mask.cpp:67-84) as MaskMatrix words."""
        seg = _i32(seg)
        L = len(seg)
        out = np.zeros((L, (L + 63) // 64), np.uint64)
        err = C.create_string_buffer(512)
        st = self.lib.vsrref_segment_mask(_ptr(seg, C.c_int), L, _ptr(out, C.c_uint64), err, 512)
        if st:
            raise OracleError(st, err.value.decode())
        return out

    def causal_mask(self, frame, lookahead: int) -> np.ndarray:
        """vsr::build_causal_mask (P/src/mask.cpp:86-101) as MaskMatrix words."""
        frame = _i32(frame)
        L = len(frame)
        out = np.zeros((L, (L + 63) // 64), np.uint64)
        err = C.create_string_buffer(512)
        st = self.lib.vsrref_causal_mask(_ptr(frame, C.c_int), L, int(lookahead), _ptr(out, C.c_uint64), err, 512)
        if st:
            raise OracleError(st, err.value.decode())
        return out

    def kv_evict(self, strategy: int, window: int, ids, scores: Optional[np.ndarray], heads: int):
        """KVCache(1, heads, window, strategy) holding `ids` on every head, then evict(0, scores)
        (P/src/kv_cache.cpp:97-137).  Returns the retained ids per head."""
        ids = _i32(ids)
        n = len(ids)
        sc = None if scores is None else np.ascontiguousarray(scores, np.float64).reshape(heads, n)
        out = np.zeros((heads, n), np.int32)
        cnt = np.zeros(heads, np.int32)
        err = C.create_string_buffer(512)
        st = self.lib.vsrref_kv_evict(strategy, heads, window, n, _ptr(ids, C.c_int),
                                      _ptr(sc, C.c_double) if sc is not None else None,
                                      _ptr(out, C.c_int), _ptr(cnt, C.c_int), err, 512)
        if st:
            raise OracleError(st, err.value.decode())
        return [list(map(int, out[h, : cnt[h]])) for h in range(heads)]

    def case(self, q, k, v, qf, kf, rows, cols, mask: Optional[Mask] = None) -> "Ref.Case":
        return Ref.Case(self.lib, q, k, v, qf, kf, rows, cols, mask or Mask.all())


# ----------------------------------------------------------------------------
# Shared helpers
# ----------------------------------------------------------------------------

def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bf16, returned as float32 (exactly representable)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) << 16
    nan = np.isnan(x)
    out = (r & 0xFFFFFFFF).astype(np.uint32).view(np.float32)
    out = np.where(nan, x, out)
    return out.astype(np.float32)


def head_scale(d: int) -> float:
    """1.0f / std::sqrt(float(d)) in fp32 (P/src/sparse.cpp:97, stream.cpp:188)."""
    return float(np.float32(1.0) / np.sqrt(np.float32(d)))


def fnv1a64(buf: bytes) -> int:
    """P/include/vsr/common.hpp:56-64."""
    h = 0xCBF29CE484222325
    for b in buf:
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def synthetic_qkv(seed: int, lq: int, lk: int, d: int, gen=None, bf16: bool = True):
    """q, k, v drawn in reference order from vsr::Rng(seed) (q first, then k, then v;
    P/src/bench.cpp:78-81), optionally rounded to bf16 so GPU and CPU see identical values."""
    gen = gen or Port()
    flat = gen.gaussian(seed, lq * d + 2 * lk * d)
    q = flat[: lq * d].reshape(lq, d)
    k = flat[lq * d: lq * d + lk * d].reshape(lk, d)
    v = flat[lq * d + lk * d:].reshape(lk, d)
    if bf16:
        q, k, v = bf16_round(q), bf16_round(k), bf16_round(v)
    return q, k, v


# ----------------------------------------------------------------------------
# Scored eviction: numpy restatement
# ----------------------------------------------------------------------------

def frame_attention_mass(plan: Plan, kf: Sequence[int], rows: int, cols: int) -> np.ndarray:
    """Per-frame attention mass of a plan over its key grid (P/src/kv_cache.cpp:170-206).

    For every q-block: softmax in double over the coarse-allowed key blocks of its fp32
    coarse scores (max, exp(s - max), sum in key-block order; rows with no allowed block are
    skipped); the per-key-block masses are summed over q-blocks in order, then each block's
    mass is split over its member tokens and credited to their frames."""
    coarse = plan.coarse.astype(np.float64)
    allowed = plan.allowed.astype(bool)
    bnq, bnk = coarse.shape
    block_mass = np.zeros(bnk, np.float64)
    for qb in range(bnq):
        if not allowed[qb].any():
            continue
        mx = coarse[qb][allowed[qb]].max()
        # math.exp is libm's exp, the function std::exp calls (numpy's SIMD exp differs in ulps)
        row = np.array([math.exp(coarse[qb, kb] - mx) if allowed[qb, kb] else 0.0 for kb in range(bnk)])
        denom = 0.0
        for x in row:  # sequential, key-block order (kv_cache.cpp:184-189)
            denom += x
        block_mass += row / denom
    assign, _ = Port().partition(kf, rows, cols)
    per_frame_tok = rows * cols
    members = np.bincount(assign, minlength=bnk).astype(np.float64)
    out = np.zeros(len(kf), np.float64)
    order = np.argsort(assign, kind="stable")  # key blocks ascending, members in token order
    for tok in order:  # (kv_cache.cpp:193-203)
        kb = assign[tok]
        if block_mass[kb] != 0.0:
            out[tok // per_frame_tok] += block_mass[kb] / members[kb]
    return out


def evict_victims(ids: Sequence[int], score: Sequence[float], excess: int):
    """Victim order for one head (P/src/kv_cache.cpp:81-93): lowest score first, older frame
    on ties, newest frame exempt."""
    idx = sorted(range(len(ids) - 1), key=lambda i: (score[i], ids[i]))
    return [int(ids[i]) for i in idx[:excess]]


def evict(strategy: int, window: int, ids: Sequence[int], scores: Optional[np.ndarray], heads: int):
    """KVCache::evict for one layer whose heads all hold `ids` (P/src/kv_cache.cpp:97-137).
    strategy 0 sliding, 1 uniform (head scores summed), 2 head-wise.  Returns retained ids per head."""
    ids = [int(i) for i in ids]
    if strategy == 0 or len(ids) <= window:
        return [ids[-window:] if len(ids) > window else list(ids) for _ in range(heads)]
    sc = np.asarray(scores, np.float64).reshape(heads, len(ids))
    if strategy == 1:
        total = np.zeros(len(ids), np.float64)
        for h in range(heads):
            total += sc[h]
        gone = set(evict_victims(ids, list(total), len(ids) - window))
        return [[i for i in ids if i not in gone] for _ in range(heads)]
    out = []
    for h in range(heads):
        gone = set(evict_victims(ids, list(sc[h]), len(ids) - window))
        out.append([i for i in ids if i not in gone])
    return out


# ----------------------------------------------------------------------------
# Token-mask builders: numpy restatement, MaskMatrix word layout
# ----------------------------------------------------------------------------

def _pack_rows(allowed: np.ndarray) -> np.ndarray:
    """bool [L][L] -> uint64 words [L][(L+63)/64], bit j%64 of word j/64 (mask.hpp:16-59)."""
    L, Lk = allowed.shape
    wpr = (Lk + 63) // 64
    pad = np.zeros((L, wpr * 64), bool)
    pad[:, :Lk] = allowed
    w = pad.reshape(L, wpr, 64).astype(np.uint64) << np.arange(64, dtype=np.uint64)
    return np.bitwise_or.reduce(w, axis=2)


def segment_mask(seg) -> np.ndarray:
    """build_segment_mask (P/src/mask.cpp:67-84): allowed iff seg[i] == seg[j]; ids must be
    >= 0 and contiguous (ConfigError otherwise)."""
    seg = np.asarray(seg, np.int64)
    if seg.size < 1:
        raise OracleError(2, "build_segment_mask: no tokens labeled")
    if (seg < 0).any():
        raise OracleError(2, "build_segment_mask: negative segment id")
    if len(np.unique(seg)) != seg.max() + 1:
        raise OracleError(2, "build_segment_mask: segment ids not contiguous")
    return _pack_rows(seg[:, None] == seg[None, :])


def causal_mask(frame, lookahead: int) -> np.ndarray:
    """build_causal_mask (P/src/mask.cpp:86-101): allowed iff frame[j] <= frame[i] + lookahead;
    frames non-decreasing, lookahead >= 0."""
    frame = np.asarray(frame, np.int64)
    if lookahead < 0:
        raise OracleError(2, "build_causal_mask: negative lookahead")
    if (np.diff(frame) < 0).any():
        raise OracleError(2, "build_causal_mask: frame indices must be non-decreasing")
    return _pack_rows(frame[None, :] <= frame[:, None] + lookahead)


# ----------------------------------------------------------------------------
# RoPE: numpy restatement of apply_rope
# ----------------------------------------------------------------------------

def apply_rope(x: np.ndarray, frame_ids: Sequence[int], rows: int, cols: int, theta0: float = 10000.0,
               axis_split=None) -> np.ndarray:
    """apply_rope (P/src/rope.cpp:30-62) at TokenGrid positions (t = absolute frame id, h, w;
    P/include/vsr/grid.hpp:74-79): per axis pair i, inv_freq = theta0^(-2i/d_axis) and
    angle = pos * inv_freq in double (libm pow/cos/sin), cos/sin rounded to float, then
    x0*c - x1*s and x0*s + x1*c in fp32 with separate multiply and add.  Default split
    RopeConfig::split_default: (d/2, d/4, d/4)."""
    x = np.asarray(x, np.float32)
    L, d = x.shape
    split = list(axis_split) if axis_split is not None else [d // 2, d // 4, d // 4]
    n = rows * cols
    tok = np.arange(L)
    pos = [np.asarray(frame_ids, np.int64)[tok // n], (tok % n) // cols, tok % cols]
    out = x.copy()
    base = 0
    for axis in range(3):
        da = split[axis]
        for i in range(da // 2):
            inv = math.pow(theta0, -2.0 * i / float(da))
            vals = np.unique(pos[axis])
            c_of = {int(p): np.float32(math.cos(1.0 * int(p) * inv)) for p in vals}
            s_of = {int(p): np.float32(math.sin(1.0 * int(p) * inv)) for p in vals}
            c = np.array([c_of[int(p)] for p in pos[axis]], np.float32)
            s = np.array([s_of[int(p)] for p in pos[axis]], np.float32)
            x0, x1 = x[:, base + 2 * i], x[:, base + 2 * i + 1]
            out[:, base + 2 * i] = (x0 * c) - (x1 * s)
            out[:, base + 2 * i + 1] = (x0 * s) + (x1 * c)
        base += da
    return out
