#!/usr/bin/env python
"""BASELINE.json configs beyond the headline bench line, through the public API (KVRing).

    python tools/configs.py [--out profiles/r1_configs.json] [--quick]

  * 1440p (90x160 latent, 240 tiles/frame, ragged bottom tile row), W=4, locality window
    72x72 (truncated and preserved) and all-allowed, k = 13.6% of the coarse-allowed blocks
  * 768x1408 two-latent chunk (Tq=2, the paper's granularity: 128-query q-blocks)
  * sparsity sweep at 768x1408, W=4: top-k 1..198 (198 = dense over the window, the
    dense-causal baseline of the same kernel) and W in {2, 4, 8}
  * the 30-layer x 32-frame stack (BASELINE config #3): attention-only time of 960 layer-
    steps extrapolated from the per-layer-step time (stated as such)

Each point: CUDA-event time of the layer-step pieces (append, mask builder, attention) from
the context's spans over `steps` steps cycling `layers` rings (inputs larger than L2), the
kernel-counted executed token pairs -> effective TFLOP/s (4*d per pair).  Synthetic N(0,1)
bf16 data.  Writes one JSON document.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import paper_2510_12747_b200 as fv  # noqa: E402
from paper_2510_12747_b200 import _abi  # noqa: E402

PEAK = 1700.6


def run_point(rows, cols, heads, d, window, topk, mask, nq=1, layers=8, steps=40, warmup=8, seed=7, rope=False):
    dev = torch.device("cuda")
    ctx = fv.Context.default()
    n = rows * cols
    gen = torch.Generator(device=dev).manual_seed(seed)
    pool = [[torch.randn((heads, nq * n if i == 0 else n, d), generator=gen, device=dev).to(torch.bfloat16)
             for i in range(3)] for _ in range(3)]
    # chunks of nq frames: W + nq slots, evict to W before each chunk
    ring = fv.KVRing(layers, heads, d, rows, cols, window + nq - 1, ctx=ctx)
    if rope:  # fused apply_rope in append (K) and the mask builder's Q pass
        ring.set_rope()
    t0 = 2 * window + 4
    for l in range(layers):
        for f in range(t0 - window, t0):
            _, k, v = pool[(f + l) % 3]
            ring.append(l, f, k, v)
            ring.evict(l, window)
    state = {"s": 0}

    def step():
        s = state["s"]
        state["s"] += 1
        l = s % layers
        t = t0 + nq * (s // layers)
        q, k, v = pool[(t + l) % 3]
        frames = list(range(t, t + nq))
        ring.evict(l, window)
        for f in frames:
            ring.append(l, f, k, v)
        ring.attention(l, q, frames, mask, topk, check_errors=False)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    ctx.check_errors()
    ctx.read_pairs()
    for kind in (_abi.TIME_APPEND, _abi.TIME_MASK_BUILDER, _abi.TIME_ATTENTION):
        ctx.timing_read(kind, clear=True)
    ctx.timing(True)
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
    ctx.timing(False)
    ctx.check_errors()
    pairs = ctx.read_pairs()
    at_ms, at_n = ctx.timing_read(_abi.TIME_ATTENTION)
    mb_ms, mb_n = ctx.timing_read(_abi.TIME_MASK_BUILDER)
    ap_ms, ap_n = ctx.timing_read(_abi.TIME_APPEND, clear=True)
    attn_us = at_ms / max(1, at_n) * 1e3
    step_us = (at_ms + mb_ms + ap_ms) / steps * 1e3
    flops = 4.0 * d * pairs / steps
    del ring
    return {"attn_us": attn_us, "mask_builder_us": mb_ms / max(1, mb_n) * 1e3,
            "append_us": ap_ms / max(1, ap_n) * 1e3, "step_us": step_us,
            "query_tokens_per_s": nq * n / (step_us * 1e-6),
            "executed_pairs_per_step": pairs / steps, "eff_tflops": flops / (attn_us * 1e-6) / 1e12,
            "frac_of_measured_bf16_peak": flops / (attn_us * 1e-6) / 1e12 / PEAK}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(os.path.dirname(HERE), "profiles", "r1_configs.json"))
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    res = {"note": "CUDA-event spans per kernel class; synthetic N(0,1) bf16; 4*d FLOP per executed pair",
           "points": []}

    def add(name, **kw):
        r = run_point(**kw)
        r.update({"name": name, **{k: (v if not isinstance(v, fv.Mask) else repr(v)) for k, v in kw.items()}})
        res["points"].append(r)
        print(json.dumps({k: r[k] for k in ("name", "attn_us", "step_us", "eff_tflops", "query_tokens_per_s")}),
              flush=True)

    all_ = fv.Mask.all_allowed()
    # headline shape and the Tq=2 chunk
    add("768x1408 W4 k27 (headline)", rows=48, cols=88, heads=12, d=128, window=4, topk=27, mask=all_)
    add("768x1408 W4 k27 fused RoPE", rows=48, cols=88, heads=12, d=128, window=4, topk=27, mask=all_, rope=True)
    add("768x1408 Tq=2 chunk W4 k36", rows=48, cols=88, heads=12, d=128, window=4, topk=36, mask=all_, nq=2)
    # 1440p
    add("1440p W4 k98 all-allowed", rows=90, cols=160, heads=12, d=128, window=4, topk=98, mask=all_, layers=4)
    add("1440p W4 k41 locality 72x72 truncated", rows=90, cols=160, heads=12, d=128, window=4, topk=41,
        mask=fv.Mask.locality(72, 72, truncated=True), layers=4)
    add("1440p W4 k41 locality 72x72 preserved", rows=90, cols=160, heads=12, d=128, window=4, topk=41,
        mask=fv.Mask.locality(72, 72, truncated=False), layers=4)
    add("768x1408 W4 k27 locality 48x72 truncated", rows=48, cols=88, heads=12, d=128, window=4, topk=27,
        mask=fv.Mask.locality(48, 72, truncated=True))
    if not args.quick:
        # sparsity sweep (198 = every block of the window: the dense-over-window baseline)
        for k in (1, 2, 4, 8, 16, 27, 32, 64, 128, 198):
            add(f"sweep 768x1408 W4 k{k}", rows=48, cols=88, heads=12, d=128, window=4, topk=k, mask=all_)
        for w, k in ((2, 18), (8, 45)):
            add(f"sweep 768x1408 W{w} k{k}", rows=48, cols=88, heads=12, d=128, window=w, topk=k, mask=all_)
    head = res["points"][0]
    res["stack_30x32"] = {"layer_steps": 960, "attention_stack_ms_extrapolated": head["step_us"] * 960 / 1e3,
                          "note": "960 layer-steps x the measured headline layer-step time (append + mask "
                                  "builder + attention), extrapolated, 1 GPU"}
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
