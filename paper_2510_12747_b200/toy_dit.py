"""The streaming toy-DiT step around the hot path (P/src/stream.cpp:198-281,
P = /root/reference/proj), on the B200.

    dit = StreamingDiT(StreamDiTConfig(...))          # ToyDiT::init shapes, random weights
    x = dit.step(x0)                                  # one latent frame through every layer

Per layer, as step() does (minus project_clip: the frame's token embedding x0 is the input):

    K, V  = rms_norm(x0, g1) @ [Wk | Wv]     one GEMM, [tokens][2D] bf16
    Q     = rms_norm(x,  g1) @ Wq            [tokens][D] bf16
    att   = ring step: KVCache::append of K/V (RoPE fused, the per-head split read in place
            from the GEMM output: fvsr_ring_step_layout), Q RoPE + mask builder + block-sparse
            attention, written as [tokens][D]
    x    += att @ Wo
    x    += silu(rms_norm(x, g2) @ W_in) @ W_out
    evict (sliding window)

rms_norm is this package's kernel (fvsr_rms_norm); the projections are plain bf16 GEMMs
(cuBLAS through torch.matmul, fp32 accumulation); the residual stream x stays fp32.  The
attention, its mask builder and the KV ring are the hot path (libfvsr_b200.so).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import List, Optional

import torch

from . import _abi
from ._abi import check
from .kv_ring import KVRing
from .sparse import Context, Mask, _stream


@dataclass
class StreamDiTConfig:
    """The StreamConfig / ToyDiT knobs the layer loop reads (P/include/vsr/stream.hpp:18-56)."""
    n_layers: int = 4
    n_heads: int = 4
    d_head: int = 64
    ffw_dim: int = 256
    latent_rows: int = 16
    latent_cols: int = 16
    window_frames: int = 4
    topk: int = 2
    mask: Optional[Mask] = None
    weight_seed: int = 1234
    rope_theta0: float = 10000.0

    @property
    def model_dim(self) -> int:
        return self.n_heads * self.d_head

    @property
    def tokens_per_frame(self) -> int:
        return self.latent_rows * self.latent_cols


@dataclass
class LayerWeights:
    """vsr::LayerWeights (P/include/vsr/stream.hpp:43-48), device-resident: bf16 GEMM operands
    ([in][out], as the reference's x @ W), fp32 RMSNorm gains; wkv = [Wk | Wv]."""
    wq: torch.Tensor
    wkv: torch.Tensor
    wo: torch.Tensor
    w_in: torch.Tensor
    w_out: torch.Tensor
    norm1_g: torch.Tensor
    norm2_g: torch.Tensor


def init_weights(cfg: StreamDiTConfig, device=None) -> List[LayerWeights]:
    """ToyDiT::init shapes and scales (P/src/stream.cpp:42-60): N(0, 0.02^2) projections, unit
    gains; torch's generator (the reference's Rng stream is not reproduced)."""
    device = device or torch.device("cuda", torch.cuda.current_device())
    g = torch.Generator(device=device).manual_seed(cfg.weight_seed)
    D, F = cfg.model_dim, cfg.ffw_dim

    def w(*shape):
        return (torch.randn(shape, generator=g, device=device) * 0.02).to(torch.bfloat16)

    layers = []
    for _ in range(cfg.n_layers):
        wq, wk, wv, wo = w(D, D), w(D, D), w(D, D), w(D, D)
        layers.append(LayerWeights(wq, torch.cat([wk, wv], dim=1).contiguous(), wo, w(D, F), w(F, D),
                                   torch.ones(D, device=device), torch.ones(D, device=device)))
    return layers


class StreamingDiT:
    """StreamState + step() of the toy DiT on the device (one layer-step per layer per frame)."""

    def __init__(self, cfg: StreamDiTConfig, weights: Optional[List[LayerWeights]] = None,
                 ctx: Optional[Context] = None):
        self.cfg = cfg
        self.ctx = ctx or Context.default()
        self.layers = weights or init_weights(cfg)
        self.mask = cfg.mask or Mask.all_allowed()
        self.ring = KVRing(cfg.n_layers, cfg.n_heads, cfg.d_head, cfg.latent_rows, cfg.latent_cols,
                           cfg.window_frames, ctx=self.ctx)
        self.ring.set_rope(cfg.rope_theta0)  # StreamConfig::rope: the default axis split
        self.t = 0
        self.scale = 1.0 / math.sqrt(cfg.d_head)
        N, D = cfg.tokens_per_frame, cfg.model_dim
        dev = self.layers[0].wq.device
        self._xn = torch.empty((N, D), dtype=torch.bfloat16, device=dev)
        self._att = torch.empty((N, D), dtype=torch.bfloat16, device=dev)
        self.trace = None  # set to a list to record per-layer intermediates (tests)

    def rms_norm(self, x: torch.Tensor, gain: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """fvsr_rms_norm: fp32 [n, D] -> bf16 [n, D]."""
        x = x.contiguous()
        out = out if out is not None else torch.empty(x.shape, dtype=torch.bfloat16, device=x.device)
        check(self.ctx.lib.fvsr_rms_norm(self.ctx.h, x.data_ptr(), gain.data_ptr(), x.shape[0], x.shape[1],
                                         out.data_ptr(), _stream()))
        return out

    def step(self, x0: torch.Tensor) -> torch.Tensor:
        """One latent frame: x0 fp32 [tokens, D] (the frame's token embedding) -> x fp32."""
        cfg = self.cfg
        N, D, d = cfg.tokens_per_frame, cfg.model_dim, cfg.d_head
        if x0.shape != (N, D) or x0.dtype != torch.float32 or not x0.is_cuda:
            raise _abi.ShapeError(f"step: x0 must be fp32 CUDA [{N}, {D}]")
        t = self.t
        x = x0.clone()
        ids = (C.c_int32 * 1)(t)
        md = self.mask.c()
        kv_lay = _abi.Layout(d, 2 * D)  # [tokens][K | V]: head h at column h*d, row stride 2D
        tok_lay = _abi.Layout(d, D)     # [tokens][D]
        for l, w in enumerate(self.layers):
            kv = self.rms_norm(x0, w.norm1_g, self._xn) @ w.wkv    # make_frame_kv (stream.cpp:134-152)
            q = self.rms_norm(x, w.norm1_g, self._xn) @ w.wq
            check(self.ctx.lib.fvsr_ring_step_layout(
                self.ctx.h, self.ring.h, l, t, kv.data_ptr(), kv[:, D:].data_ptr(), kv_lay, q.data_ptr(), tok_lay,
                ids, 1, C.byref(md), int(cfg.topk), float(self.scale), self._att.data_ptr(), tok_lay, _stream()))
            self.ring.evict(l)
            if self.trace is not None:
                self.trace.append({"layer": l, "x": x.clone(), "kv": kv.clone(), "q": q.clone(),
                                   "att": self._att.clone()})
            x += (self._att @ w.wo).float()                        # stream.cpp:257
            h1 = torch.nn.functional.silu((self.rms_norm(x, w.norm2_g, self._xn) @ w.w_in).float())
            x += (h1.to(torch.bfloat16) @ w.w_out).float()          # stream.cpp:258-259
        self.t = t + 1
        return x
