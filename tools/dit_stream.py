#!/usr/bin/env python
"""End-to-end streaming throughput of the toy DiT around the hot path at the paper's shape
(BASELINE config #3: 768x1408 -> 48x88 latent, 12 heads x d 128, 30 layers, ffw 4D, W=4,
top-k 27): latent frames/s on one B200 through paper_2510_12747_b200.toy_dit (RMSNorm kernel,
cuBLAS bf16 projections, fused ring append / mask builder / sparse attention), plus the
attention share from the library's CUDA-event spans.  Synthetic N(0,1) frame embeddings,
random ToyDiT::init-scaled weights; project_clip (LR encoder) excluded.

    python tools/dit_stream.py [--frames 12] [--layers 30] [--out profiles/r2_dit_stream.json]
"""
import argparse
import json
import os
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import paper_2510_12747_b200 as fv  # noqa: E402
from paper_2510_12747_b200 import _abi  # noqa: E402
from paper_2510_12747_b200.toy_dit import StreamDiTConfig, StreamingDiT  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=12)
    ap.add_argument("--warmup", type=int, default=6)
    ap.add_argument("--layers", type=int, default=30)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    cfg = StreamDiTConfig(n_layers=args.layers, n_heads=12, d_head=128, ffw_dim=4 * 1536, latent_rows=48,
                          latent_cols=88, window_frames=4, topk=27)
    dit = StreamingDiT(cfg)
    ctx = dit.ctx
    N, D = cfg.tokens_per_frame, cfg.model_dim
    gen = torch.Generator(device="cuda").manual_seed(1)
    frames = [torch.randn((N, D), generator=gen, device="cuda") for _ in range(4)]
    for i in range(args.warmup):
        dit.step(frames[i % 4])
    torch.cuda.synchronize()
    ctx.check_errors()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(args.frames):
        dit.step(frames[i % 4])
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.frames
    # attention share: a second pass with per-class spans
    ctx.timing_read(_abi.TIME_ATTENTION, clear=True)
    ctx.timing(True)
    for i in range(args.frames):
        dit.step(frames[i % 4])
    torch.cuda.synchronize()
    ctx.timing(False)
    at_ms, at_n = ctx.timing_read(_abi.TIME_ATTENTION)
    fr_ms, fr_n = ctx.timing_read(_abi.TIME_FRONT, clear=True)
    gemm_flops = cfg.n_layers * (2 * N * D * (4 * D) + 2 * 2 * N * D * cfg.ffw_dim)
    res = {"what": "toy-DiT streaming step (stream.cpp:198-281 minus project_clip), 1 B200",
           "config": {"latent": [48, 88], "heads": 12, "d_head": 128, "layers": cfg.n_layers, "ffw": cfg.ffw_dim,
                      "window": 4, "topk": 27, "mask": "all"},
           "ms_per_latent_frame": ms, "latent_frames_per_s": 1e3 / ms, "lr_fps_x4": 4e3 / ms,
           "attention_ms_per_frame": at_ms / args.frames, "front_ms_per_frame": fr_ms / args.frames,
           "projection_ffn_gemm_tflop_per_frame": gemm_flops / 1e12,
           "note": "attention/front from CUDA-event spans in a second pass; frames/s from events around the loop"}
    print(json.dumps(res))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
