"""Device-resident ring-buffer KV cache for chunk-by-chunk streaming.

Replaces vsr::KVCache (P/include/vsr/kv_cache.hpp:27-73; P = /root/reference/proj) with
the sliding-window strategy, plus the per-step ``concat_rows`` context assembly of
step() (P/src/stream.cpp:244-249): a layer keeps window+1 frame slots per head in HBM,
tile-major and pre-swizzled for the tensor-core kernel, and attention addresses the
slots directly, so no context is ever copied.

    ring = KVRing(layers, heads, d, rows, cols, window_frames)
    ring.append(layer, t, k, v)             # KVCache::append for every head
    out  = ring.attention(layer, q, [t], mask, topk)   # head_attention, all heads
    ring.evict(layer)                       # KVCache::evict (sliding window)

Scored eviction (P/src/kv_cache.cpp:97-137, 170-206): right after ``attention``,
``mass = ring.frame_mass(layer, [t], mask)`` gives head_attention's frame_scores from the
coarse scores the mask builder left on the device, and
``ring.evict_scored(layer, EVICT_UNIFORM, mass)`` applies KVCache::evict(uniform).
"""
from __future__ import annotations

import ctypes as C
import math
from typing import Optional, Sequence

import torch

from . import _abi
from ._abi import ShapeError, check
from .sparse import Context, Mask, _heads3, _stream


EVICT_SLIDING, EVICT_UNIFORM, EVICT_HEAD_WISE = 0, 1, 2  # vsr::EvictStrategy (kv_cache.hpp:12)


class KVRing:
    def __init__(self, layers: int, heads: int, d: int, rows: int, cols: int, window_frames: int,
                 ctx: Optional[Context] = None):
        self.ctx = ctx or Context.default()
        self.layers, self.heads, self.d, self.rows, self.cols = layers, heads, d, rows, cols
        self.window = window_frames
        h = C.c_void_p()
        check(self.ctx.lib.fvsr_ring_create(self.ctx.h, layers, heads, d, rows, cols, window_frames, C.byref(h)))
        self.h = h
        self._last_mask = {}  # layer -> mask of the last attention call (frame_mass default)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.ctx.lib.fvsr_ring_destroy(self.h)
        except Exception:
            pass

    @property
    def tokens_per_frame(self) -> int:
        return self.rows * self.cols

    def _frame(self, x: torch.Tensor, name: str) -> torch.Tensor:
        x3 = _heads3(x, name)
        if x3.shape != (self.heads, self.tokens_per_frame, self.d):
            raise ShapeError(f"{name}: expected [{self.heads}, {self.tokens_per_frame}, {self.d}], got {tuple(x3.shape)}")
        return x3

    def append(self, layer: int, frame_id: int, k: torch.Tensor, v: torch.Tensor) -> None:
        k3, v3 = self._frame(k, "append k"), self._frame(v, "append v")
        check(self.ctx.lib.fvsr_ring_append(self.ctx.h, self.h, layer, int(frame_id), k3.data_ptr(), v3.data_ptr(),
                                            _stream()))

    def set_rope(self, theta0: float = 10000.0, axis_split: Optional[Sequence[int]] = None) -> None:
        """Fuse apply_rope (P/src/rope.cpp:30-62) into the ring: append rotates K and attention
        rotates Q at absolute (frame, row, col) positions; inputs become un-rotated projections."""
        sp = None if axis_split is None else (C.c_int32 * 3)(*[int(a) for a in axis_split])
        check(self.ctx.lib.fvsr_ring_set_rope(self.h, float(theta0), sp))

    def evict(self, layer: int, keep: Optional[int] = None) -> None:
        """KVCache::evict(sliding): down to the window, or to `keep` frames (chunked streaming)."""
        if keep is None:
            check(self.ctx.lib.fvsr_ring_evict_sliding(self.h, layer))
        else:
            check(self.ctx.lib.fvsr_ring_evict_keep(self.h, layer, int(keep)))

    def frame_mass(self, layer: int, q_frame_ids: Sequence[int], mask: Optional[Mask] = None,
                   check_errors: bool = True) -> torch.Tensor:
        """frame_attention_mass of the plan of the preceding ``attention`` call on this
        layer (same q frames and mask): float64 [heads, retained frames] on the device.  The
        mask defaults to that call's; the library refuses scores of any other call."""
        mask = mask or self._last_mask.get(layer) or Mask.all_allowed()
        nq = len(q_frame_ids)
        ids = (C.c_int32 * nq)(*[int(f) for f in q_frame_ids])
        md = mask.c()
        mass = torch.empty((self.heads, self.retained(layer)), dtype=torch.float64,
                           device=torch.device("cuda", torch.cuda.current_device()))
        check(self.ctx.lib.fvsr_ring_frame_mass(self.ctx.h, self.h, layer, ids, nq, C.byref(md), mass.data_ptr(),
                                                _stream()))
        if check_errors:
            self.ctx.check_errors()
        return mass

    def evict_scored(self, layer: int, strategy: int, scores=None) -> None:
        """KVCache::evict(layer, scores) (P/src/kv_cache.cpp:97-137); scores [heads, frames]
        aligned with frame_ids (a device tensor is copied to the host first)."""
        buf = None
        if scores is not None:
            t = torch.as_tensor(scores, dtype=torch.float64).detach().cpu().contiguous()
            if t.shape != (self.heads, self.retained(layer)):
                raise ShapeError("KVCache: score count must match retained frames")
            buf = t
        check(self.ctx.lib.fvsr_ring_evict(self.h, layer, int(strategy), buf.data_ptr() if buf is not None else None))

    def frame_ids(self, layer: int):
        buf = (C.c_int32 * 64)()
        n = C.c_int32()
        check(self.ctx.lib.fvsr_ring_frame_ids(self.h, layer, buf, 64, C.byref(n)))
        return [buf[i] for i in range(n.value)]

    def frame_ids_head(self, layer: int, head: int):
        """Frames head `head` of `layer` retains (head-wise eviction lets heads diverge)."""
        buf = (C.c_int32 * 64)()
        n = C.c_int32()
        check(self.ctx.lib.fvsr_ring_frame_ids_head(self.h, layer, head, buf, 64, C.byref(n)))
        return [buf[i] for i in range(n.value)]

    def retained(self, layer: int) -> int:
        return len(self.frame_ids(layer))

    def attention(self, layer: int, q: torch.Tensor, q_frame_ids: Sequence[int], mask: Optional[Mask] = None,
                  topk: int = 1, scale: Optional[float] = None, *, unit_begin: int = 0, unit_end: int = -1,
                  out: Optional[torch.Tensor] = None, tile_major: bool = False,
                  sel: Optional[torch.Tensor] = None, sel_count: Optional[torch.Tensor] = None,
                  check_errors: bool = True, _append=None) -> torch.Tensor:
        mask = mask or Mask.all_allowed()
        self._last_mask[layer] = mask
        q3 = _heads3(q, "ring attention q")
        nq = len(q_frame_ids)
        if q3.shape != (self.heads, nq * self.tokens_per_frame, self.d):
            raise ShapeError("ring attention: q must be [heads, nq*rows*cols, d]")
        if scale is None:
            scale = 1.0 / math.sqrt(self.d)
        if out is None:
            if tile_major:
                from .head_parallel import unit_space
                ntr, fpu = unit_space(q_frame_ids)
                tiles = ((self.rows + 7) // 8) * ((self.cols + 7) // 8)
                total = self.heads * ntr * tiles
                u1 = total if unit_end < 0 else min(unit_end, total)
                out = torch.empty(((u1 - unit_begin), 64 * fpu, self.d), dtype=torch.bfloat16, device=q3.device)
            else:
                out = torch.empty_like(q3)
        ids = (C.c_int32 * nq)(*[int(f) for f in q_frame_ids])
        md = mask.c()
        cap = sel.shape[-1] if sel is not None else 0
        sp = sel.data_ptr() if sel is not None else None
        cp = sel_count.data_ptr() if sel_count is not None else None
        if _append is None:
            check(self.ctx.lib.fvsr_ring_attention(self.ctx.h, self.h, layer, q3.data_ptr(), ids, nq, C.byref(md),
                                                   int(topk), float(scale), int(unit_begin), int(unit_end),
                                                   out.data_ptr(), 1 if tile_major else 0, cap, sp, cp, _stream()))
        else:
            fid, k3, v3 = _append
            check(self.ctx.lib.fvsr_ring_step(self.ctx.h, self.h, layer, fid, k3.data_ptr(), v3.data_ptr(),
                                              q3.data_ptr(), ids, nq, C.byref(md), int(topk), float(scale),
                                              int(unit_begin), int(unit_end), out.data_ptr(), 1 if tile_major else 0,
                                              cap, sp, cp, _stream()))
        if check_errors:
            self.ctx.check_errors()
        return out

    def step(self, layer: int, frame_id: int, k: torch.Tensor, v: torch.Tensor, q: torch.Tensor,
             q_frame_ids: Optional[Sequence[int]] = None, mask: Optional[Mask] = None, topk: int = 1,
             scale: Optional[float] = None, *, unit_begin: int = 0, unit_end: int = -1,
             out: Optional[torch.Tensor] = None, tile_major: bool = False, sel: Optional[torch.Tensor] = None,
             sel_count: Optional[torch.Tensor] = None, check_errors: bool = True) -> torch.Tensor:
        """append(layer, frame_id, k, v) + attention(layer, q, q_frame_ids, ...) as ONE C-ABI call
        (fvsr_ring_step): the append and the mask builder share one kernel launch."""
        k3, v3 = self._frame(k, "append k"), self._frame(v, "append v")
        q_frame_ids = [int(frame_id)] if q_frame_ids is None else [int(f) for f in q_frame_ids]
        return self.attention(layer, q, q_frame_ids, mask, topk, scale, unit_begin=unit_begin, unit_end=unit_end,
                              out=out, tile_major=tile_major, sel=sel, sel_count=sel_count,
                              check_errors=check_errors, _append=(int(frame_id), k3, v3))

    def step_host(self, layer: int, frame_id: int, q_host: torch.Tensor, k_host: torch.Tensor,
                  v_host: torch.Tensor, out_host: torch.Tensor, mask: Optional[Mask] = None, topk: int = 1,
                  scale: Optional[float] = None) -> None:
        """One streaming layer-step from host (pinned) bf16 buffers: H2D, append, attention,
        sliding evict, D2H.  Asynchronous on the current stream."""
        mask = mask or Mask.all_allowed()
        for t, nm in ((q_host, "q"), (k_host, "k"), (v_host, "v"), (out_host, "out")):
            if t.is_cuda or t.dtype != torch.bfloat16 or t.numel() != self.heads * self.tokens_per_frame * self.d:
                raise ShapeError(f"step_host {nm}: host bf16 tensor of heads*rows*cols*d elements required")
        if scale is None:
            scale = 1.0 / math.sqrt(self.d)
        md = mask.c()
        check(self.ctx.lib.fvsr_ring_step_host(self.ctx.h, self.h, layer, int(frame_id), q_host.data_ptr(),
                                               k_host.data_ptr(), v_host.data_ptr(), C.byref(md), int(topk),
                                               float(scale), out_host.data_ptr(), _stream()))
