"""Python mirror of the reference's block-sparse operator API, on B200 device tensors.

Same names, argument meaning and error behaviour as P/include/vsr/sparse.hpp:16-66
(P = /root/reference/proj); the work happens in libfvsr_b200.so through the C-ABI
(include/fvsr_b200.h).  torch is used only for device memory and the current stream.

    plan = plan_sparse(q, k, grid_q, grid_k, mask, topk)      # sparse.hpp:45-52
    out  = sparse_attention_exec(q, k, v, plan, mask, scale)  # sparse.hpp:59-64
    rep  = sparsity_report(plan, mask)                        # sparse.hpp:66

Tensors are bf16 CUDA tensors, [L, d] for one head or [heads, L, d].
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import torch

from . import _abi
from ._abi import (MASK_ALL, MASK_BITMASK, MASK_LOCALITY, LOCALITY_PRESERVED, LOCALITY_TRUNCATED, ConfigError,
                   ShapeError, check)


# ---------------------------------------------------------------------------------------
# value types
# ---------------------------------------------------------------------------------------

@dataclass(frozen=True)
class TokenGrid:
    """vsr::TokenGrid (P/include/vsr/grid.hpp:22-46): absolute frame ids over rows x cols."""
    frame_ids: tuple
    rows: int
    cols: int

    def __init__(self, frame_ids, rows: int, cols: int):
        if isinstance(frame_ids, int):  # contiguous 0..n-1 constructor (grid.hpp:29)
            frame_ids = tuple(range(frame_ids))
        object.__setattr__(self, "frame_ids", tuple(int(f) for f in frame_ids))
        object.__setattr__(self, "rows", int(rows))
        object.__setattr__(self, "cols", int(cols))

    def token_count(self) -> int:
        return len(self.frame_ids) * self.rows * self.cols

    def frame_count(self) -> int:
        return len(self.frame_ids)

    def tokens_per_frame(self) -> int:
        return self.rows * self.cols

    def c(self):
        return _abi.make_grid(self.frame_ids, self.rows, self.cols)


@dataclass(frozen=True)
class Mask:
    """Token mask: all-allowed, locality window (analytic), or explicit MaskMatrix bits.

    == vsr::MaskMatrix::all_allowed / build_locality_mask / MaskMatrix (P/include/vsr/mask.hpp)."""
    kind: int = MASK_ALL
    mode: int = LOCALITY_TRUNCATED
    extent_h: int = 1
    extent_w: int = 1
    bits: Optional[torch.Tensor] = None  # int64 CUDA tensor [Lq, words_per_row] (uint64 bit patterns)

    @staticmethod
    def all_allowed() -> "Mask":
        return Mask(MASK_ALL)

    @staticmethod
    def locality(extent_h: int, extent_w: int, truncated: bool = True) -> "Mask":
        return Mask(MASK_LOCALITY, LOCALITY_TRUNCATED if truncated else LOCALITY_PRESERVED, int(extent_h),
                    int(extent_w))

    @staticmethod
    def bitmask(bits: torch.Tensor) -> "Mask":
        if bits.dtype not in (torch.int64, torch.uint64) or not bits.is_cuda or bits.dim() != 2:
            raise ShapeError("bitmask must be a 2-D int64/uint64 CUDA tensor [Lq, words_per_row]")
        return Mask(MASK_BITMASK, 0, 1, 1, bits.contiguous())

    def c(self):
        if self.kind == MASK_BITMASK:
            return _abi.MaskDesc(MASK_BITMASK, 0, 1, 1, self.bits.data_ptr(), self.bits.shape[1])
        return _abi.MaskDesc(self.kind, self.mode, self.extent_h, self.extent_w, None, 0)


@dataclass
class SparsePlan:
    """vsr::SparsePlan (P/include/vsr/sparse.hpp:16-29), device-resident, per head."""
    topk: int
    head_dim: int
    grid_q: TokenGrid
    grid_k: TokenGrid
    sel: torch.Tensor            # int32 [heads, bnq, cap], ascending, -1 padded
    count: torch.Tensor          # int32 [heads, bnq]
    diagonal_block: torch.Tensor # int32 [heads, bnq]
    coarse_scores: Optional[torch.Tensor] = None   # float32 [heads, bnq, bnk]
    coarse_allowed: Optional[torch.Tensor] = None  # uint8 [heads, bnq, bnk]
    mask: Optional["Mask"] = None                  # the token mask the plan was built with

    @property
    def heads(self) -> int:
        return self.sel.shape[0]

    @property
    def bnq(self) -> int:
        return self.sel.shape[1]

    def selected(self, head: int = 0) -> List[List[int]]:
        s, n = self.sel[head].cpu(), self.count[head].cpu()
        return [s[i, : int(n[i])].tolist() for i in range(s.shape[0])]

    def selected_pairs(self) -> int:
        return int(self.count.sum().item())


@dataclass
class SparsityReport:
    """vsr::SparsityReport (P/include/vsr/sparse.hpp:33-38), summed over heads."""
    density: float
    executed_flops: int
    dense_flops: int
    flop_ratio: float
    executed_pairs: int = 0
    per_head_executed_pairs: List[int] = field(default_factory=list)


# ---------------------------------------------------------------------------------------
# context
# ---------------------------------------------------------------------------------------

class Context:
    """Owns an fvsr_ctx (device error word + workspace) on the current CUDA device."""

    _per_device = {}

    def __init__(self):
        self.lib = _abi.load()
        h = C.c_void_p()
        check(self.lib.fvsr_ctx_create(C.byref(h)))
        self.h = h
        self.device = torch.cuda.current_device()

    @classmethod
    def default(cls) -> "Context":
        dev = torch.cuda.current_device()
        if dev not in cls._per_device:
            cls._per_device[dev] = Context()
        return cls._per_device[dev]

    def check_errors(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        s = (stream or torch.cuda.current_stream()).cuda_stream
        check(self.lib.fvsr_check_errors(self.h, C.c_void_p(s)))

    def launch_count(self) -> int:
        return int(self.lib.fvsr_ctx_launch_count(self.h))

    def set_flags(self, flags: int) -> None:
        """fvsr_ctx_set_flags: FLAG_SYNC_CHECK | FLAG_NO_TMA (see include/fvsr_b200.h)."""
        self.flags = int(flags)
        check(self.lib.fvsr_ctx_set_flags(self.h, int(flags)))

    def timing(self, enable: bool) -> None:
        check(self.lib.fvsr_ctx_timing_enable(self.h, 1 if enable else 0))

    def timing_read(self, kind: int, clear: bool = False):
        ms, n = C.c_double(), C.c_int64()
        check(self.lib.fvsr_ctx_timing_read(self.h, kind, C.byref(ms), C.byref(n), 1 if clear else 0))
        return ms.value, n.value

    def read_pairs(self) -> int:
        v = C.c_uint64()
        check(self.lib.fvsr_ctx_read_pairs(self.h, C.byref(v)))
        return v.value

    def read_tiles(self):
        """(key tiles issued, of them with 128 key rows) since the last read; resets."""
        t, f = C.c_uint64(), C.c_uint64()
        check(self.lib.fvsr_ctx_read_tiles(self.h, C.byref(t), C.byref(f)))
        return t.value, f.value

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.fvsr_ctx_destroy(self.h)
        except Exception:
            pass


def _stream() -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _heads3(x: torch.Tensor, name: str, fp32_ok: bool = False) -> torch.Tensor:
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise ShapeError(f"{name}: CUDA tensor required")
    if x.dtype != torch.bfloat16 and not (fp32_ok and x.dtype == torch.float32):
        raise ShapeError(f"{name}: bf16 tensor required (got {x.dtype})")
    if x.dim() == 2:
        x = x.unsqueeze(0)
    if x.dim() != 3:
        raise ShapeError(f"{name}: rank-2 [L, d] or rank-3 [heads, L, d] operand required")
    return x.contiguous()


def block_counts(grid_q: TokenGrid, grid_k: TokenGrid):
    lib = _abi.load()
    gq, kq = grid_q.c()
    gk, kk = grid_k.c()
    bnq, bnk = C.c_int32(), C.c_int32()
    check(lib.fvsr_block_counts(C.byref(gq), C.byref(gk), C.byref(bnq), C.byref(bnk)))
    return bnq.value, bnk.value


# ---------------------------------------------------------------------------------------
# operators
# ---------------------------------------------------------------------------------------

def plan_sparse(q: torch.Tensor, k: torch.Tensor, grid_q: TokenGrid, grid_k: Optional[TokenGrid] = None,
                mask: Optional[Mask] = None, topk: int = 1, *, keep_scores: bool = True,
                ctx: Optional[Context] = None, check_errors: bool = True) -> SparsePlan:
    """plan_sparse (P/src/sparse.cpp:72-139); self form when grid_k is None."""
    ctx = ctx or Context.default()
    grid_k = grid_k or grid_q
    mask = mask or Mask.all_allowed()
    q3, k3 = _heads3(q, "plan_sparse q", fp32_ok=True), _heads3(k, "plan_sparse k", fp32_ok=True)
    if q3.shape[0] != k3.shape[0] or q3.shape[2] != k3.shape[2]:
        raise ShapeError("plan_sparse: q/k dim mismatch")
    if q3.shape[1] != grid_q.token_count() or k3.shape[1] != grid_k.token_count():
        raise ShapeError("plan_sparse: partitions do not cover the inputs")
    if mask.kind == MASK_BITMASK and mask.bits.shape[0] != grid_q.token_count():
        raise ShapeError("plan_sparse: mask shape mismatch")
    heads, d = q3.shape[0], q3.shape[2]
    if int(topk) < 1:
        raise ConfigError("plan_sparse: topk must be >= 1")
    bnq, bnk = block_counts(grid_q, grid_k)
    cap = max(1, min(int(topk), bnk))
    dev = q3.device
    sel = torch.empty((heads, bnq, cap), dtype=torch.int32, device=dev)
    cnt = torch.empty((heads, bnq), dtype=torch.int32, device=dev)
    diag = torch.empty((heads, bnq), dtype=torch.int32, device=dev)
    coarse = torch.empty((heads, bnq, bnk), dtype=torch.float32, device=dev) if keep_scores else None
    allowed = torch.empty((heads, bnq, bnk), dtype=torch.uint8, device=dev) if keep_scores else None
    gq, kq = grid_q.c()
    gk, kk = grid_k.c()
    md = mask.c()
    if q3.dtype != k3.dtype:
        raise ShapeError("plan_sparse: q and k must have the same dtype")
    # fp32 inputs (the reference's own) are pooled as they are: the plan is bit-exact with
    # vsr::plan_sparse on any data; bf16 inputs are the streaming path's
    fn = ctx.lib.fvsr_plan_sparse_f32 if q3.dtype == torch.float32 else ctx.lib.fvsr_plan_sparse
    check(fn(ctx.h, q3.data_ptr(), k3.data_ptr(), heads, d, C.byref(gq), C.byref(gk),
             C.byref(md), int(topk), cap, sel.data_ptr(), cnt.data_ptr(), diag.data_ptr(),
             coarse.data_ptr() if coarse is not None else None,
             allowed.data_ptr() if allowed is not None else None, _stream()))
    if check_errors:
        ctx.check_errors()
    return SparsePlan(int(topk), d, grid_q, grid_k, sel, cnt, diag, coarse, allowed, mask)


def sparse_attention_exec(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, plan: SparsePlan,
                          mask: Optional[Mask] = None, scale: Optional[float] = None, row_begin: int = 0,
                          row_end: Optional[int] = None, *, out: Optional[torch.Tensor] = None,
                          ctx: Optional[Context] = None, check_errors: bool = True) -> torch.Tensor:
    """sparse_attention_exec (P/src/sparse.cpp:208-254) on tcgen05; returns bf16 like q."""
    ctx = ctx or Context.default()
    mask = mask or Mask.all_allowed()
    squeeze = q.dim() == 2
    q3, k3, v3 = _heads3(q, "exec q"), _heads3(k, "exec k"), _heads3(v, "exec v")
    if k3.shape != v3.shape:
        raise ShapeError("sparse_attention_exec: plan does not match inputs")
    if q3.shape[1] != plan.grid_q.token_count() or k3.shape[1] != plan.grid_k.token_count():
        raise ShapeError("sparse_attention_exec: plan does not match inputs")
    if q3.shape[2] != k3.shape[2] or q3.shape[2] != plan.head_dim:
        raise ShapeError("sparse_attention_exec: head dim mismatch")
    if q3.shape[0] != plan.heads or k3.shape[0] != plan.heads:
        raise ShapeError("sparse_attention_exec: head count mismatch")
    heads, lq, d = q3.shape
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    if out is None:
        out = torch.empty_like(q3)
    gq, kq = plan.grid_q.c()
    gk, kk = plan.grid_k.c()
    md = mask.c()
    check(ctx.lib.fvsr_sparse_attention_exec(ctx.h, q3.data_ptr(), k3.data_ptr(), v3.data_ptr(), heads, d,
                                             C.byref(gq), C.byref(gk), C.byref(md), plan.sel.shape[2],
                                             plan.sel.data_ptr(), plan.count.data_ptr(), float(scale),
                                             int(row_begin), -1 if row_end is None else int(row_end),
                                             out.data_ptr(), _stream()))
    if check_errors:
        ctx.check_errors()
    return out[0] if squeeze else out


def _labels(x, name):
    a = torch.as_tensor(x).detach().to("cpu", torch.int32).contiguous()
    if a.dim() != 1:
        raise ShapeError(f"{name}: labels must be 1-D")
    return a


def build_segment_mask(seg, *, ctx: Optional[Context] = None, device=None) -> Mask:
    """build_segment_mask (P/src/mask.cpp:67-84) on device -> a bitmask Mask (Lq = Lk = L)."""
    ctx = ctx or Context.default()
    lab = _labels(seg, "build_segment_mask")
    L = lab.numel()
    bits = torch.empty((max(L, 1), (L + 63) // 64 or 1), dtype=torch.int64,
                       device=device or torch.device("cuda", torch.cuda.current_device()))
    check(ctx.lib.fvsr_build_segment_mask(ctx.h, C.cast(lab.data_ptr(), C.POINTER(C.c_int32)), L, bits.data_ptr(),
                                          _stream()))
    return Mask.bitmask(bits)


def build_causal_mask(frame, lookahead: int = 0, *, ctx: Optional[Context] = None, device=None) -> Mask:
    """build_causal_mask (P/src/mask.cpp:86-101) on device -> a bitmask Mask."""
    ctx = ctx or Context.default()
    lab = _labels(frame, "build_causal_mask")
    L = lab.numel()
    bits = torch.empty((max(L, 1), (L + 63) // 64 or 1), dtype=torch.int64,
                       device=device or torch.device("cuda", torch.cuda.current_device()))
    check(ctx.lib.fvsr_build_causal_mask(ctx.h, C.cast(lab.data_ptr(), C.POINTER(C.c_int32)), L, int(lookahead),
                                         bits.data_ptr(), _stream()))
    return Mask.bitmask(bits)


def _same_mask(a: "Mask", b: "Mask") -> bool:
    if a.kind != b.kind:
        return False
    if a.kind == MASK_ALL:
        return True
    if a.kind == MASK_LOCALITY:
        return (a.mode, a.extent_h, a.extent_w) == (b.mode, b.extent_h, b.extent_w)
    return a.bits is b.bits or (a.bits.shape == b.bits.shape and bool(torch.equal(a.bits, b.bits)))


def frame_attention_mass(plan: SparsePlan, key_grid: Optional[TokenGrid] = None, mask: Optional[Mask] = None, *,
                         ctx: Optional[Context] = None, check_errors: bool = True) -> torch.Tensor:
    """frame_attention_mass (P/src/kv_cache.cpp:170-206) on device: float64 [heads, frames]
    of key_grid (default plan.grid_k).  The coarse-allowed blocks are the plan's own, as in
    the reference (kv_cache.cpp:177-188): the mask defaults to the one the plan was built with,
    and a different one is refused.  The plan must keep its coarse scores."""
    ctx = ctx or Context.default()
    own = plan.mask or Mask.all_allowed()
    if mask is not None and not _same_mask(mask, own):
        raise ConfigError("frame_attention_mass: mask differs from the one the plan was built with")
    mask = own
    key_grid = key_grid or plan.grid_k
    if plan.coarse_scores is None:
        raise ConfigError("frame_attention_mass: plan was built without coarse scores (keep_scores=False)")
    if key_grid.token_count() != plan.grid_k.token_count():
        raise ShapeError("frame_attention_mass: plan does not match key grid")
    mass = torch.empty((plan.heads, key_grid.frame_count()), dtype=torch.float64, device=plan.coarse_scores.device)
    gq, kq = plan.grid_q.c()
    gk, kk = key_grid.c()
    md = mask.c()
    check(ctx.lib.fvsr_frame_attention_mass(ctx.h, plan.heads, C.byref(gq), C.byref(gk), C.byref(md),
                                            plan.coarse_scores.data_ptr(), mass.data_ptr(), _stream()))
    if check_errors:
        ctx.check_errors()
    return mass


def sparsity_report(plan: SparsePlan, mask: Optional[Mask] = None, *, ctx: Optional[Context] = None) -> SparsityReport:
    """sparsity_report (P/src/sparse.cpp:256-285), summed over heads."""
    ctx = ctx or Context.default()
    mask = mask or Mask.all_allowed()
    heads = plan.heads
    dev = plan.sel.device
    outs = [torch.zeros(heads, dtype=torch.int64, device=dev) for _ in range(4)]
    gq, kq = plan.grid_q.c()
    gk, kk = plan.grid_k.c()
    md = mask.c()
    check(ctx.lib.fvsr_sparsity_report(ctx.h, heads, C.byref(gq), C.byref(gk), C.byref(md), plan.sel.shape[2],
                                       plan.sel.data_ptr(), plan.count.data_ptr(), *[o.data_ptr() for o in outs],
                                       _stream()))
    ex, dense, nsel, nallow = [o.cpu().tolist() for o in outs]
    if sum(nallow) == 0:
        raise _abi.InvariantError("sparsity_report: no allowed block pairs")
    per_pair = 2 * plan.head_dim + 2
    return SparsityReport(density=sum(nsel) / sum(nallow), executed_flops=sum(ex) * per_pair,
                          dense_flops=sum(dense) * per_pair,
                          flop_ratio=(sum(ex) / sum(dense)) if sum(dense) else 0.0,
                          executed_pairs=sum(ex), per_head_executed_pairs=ex)
