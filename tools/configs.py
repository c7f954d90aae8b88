#!/usr/bin/env python
"""BASELINE.json configs beyond the headline bench line, through the public API (KVRing).

    python tools/configs.py [--out profiles/r2_configs.json] [--quick]

  * 1440p (90x160 latent, 240 tiles/frame, ragged bottom tile row), W=4, locality window
    72x72 (truncated and preserved) and all-allowed, k = 13.6% of the coarse-allowed blocks
  * 768x1408 two-latent chunk (Tq=2, the paper's granularity: 128-query q-blocks)
  * sparsity sweep at 768x1408, W=4: top-k 1..198 (198 = dense over the window, the
    dense-causal baseline of the same kernel) and W in {2, 4, 8}
  * the 30-layer x 32-frame stack (BASELINE config #3): attention-only time of 960 layer-
    steps extrapolated from the per-layer-step time (stated as such)

Each point: the layer-step through fvsr_ring_step (ring append + mask builder + attention)
over `steps` steps cycling `layers` rings (inputs larger than L2): the step time from CUDA
events around the whole loop, then per-kernel-class spans (front = append + mask builder,
attention) in a second pass (span events serialise the programmatic launch overlap), the
kernel-counted executed token pairs -> effective TFLOP/s (4*d per pair) against the measured
bf16 peak (MEASURED_PEAKS.json).  Also the reference's dense baseline dense_attention_stream
(P/src/attention.cpp:58-99) timed on a bounded CPU sample and extrapolated (stated so).
Synthetic N(0,1) bf16 data.  Writes one JSON document.
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

def _peak():
    try:
        with open(os.path.join(os.path.dirname(HERE), "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops"]), "MEASURED_PEAKS.json bf16_tflops (burst)"
    except Exception:
        return 1590.0, "fallback (B200_PROFILING.md)"


PEAK, PEAK_SRC = _peak()


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
        for f in frames[:-1]:
            ring.append(l, f, k, v)
        ring.step(l, frames[-1], k, v, q, frames, mask, topk, check_errors=False)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    ctx.check_errors()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        step()
    b.record()
    torch.cuda.synchronize()
    step_us = a.elapsed_time(b) / steps * 1e3
    ctx.read_pairs()
    for kind in (_abi.TIME_APPEND, _abi.TIME_FRONT, _abi.TIME_ATTENTION):
        ctx.timing_read(kind, clear=True)
    ctx.timing(True)
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
    ctx.timing(False)
    ctx.check_errors()
    pairs = ctx.read_pairs()
    at_ms, at_n = ctx.timing_read(_abi.TIME_ATTENTION)
    fr_ms, fr_n = ctx.timing_read(_abi.TIME_FRONT)
    ap_ms, ap_n = ctx.timing_read(_abi.TIME_APPEND, clear=True)
    attn_us = at_ms / max(1, at_n) * 1e3
    flops = 4.0 * d * pairs / steps
    del ring
    return {"attn_us": attn_us, "front_us": fr_ms / max(1, fr_n) * 1e3,
            "extra_append_us": ap_ms / max(1, ap_n) * 1e3 if ap_n else 0.0, "step_us": step_us,
            "query_tokens_per_s": nq * n / (step_us * 1e-6),
            "executed_pairs_per_step": pairs / steps, "eff_tflops": flops / (attn_us * 1e-6) / 1e12,
            "frac_of_measured_bf16_peak": flops / (attn_us * 1e-6) / 1e12 / PEAK}


def cpu_dense_stream(rows=48, cols=88, d=128, window=4, heads=12, sample_rows=64):
    """The reference's dense baseline (dense_attention_stream) per head at the streaming step,
    timed on `sample_rows` query rows and extrapolated to the layer-step (12 heads)."""
    import time
    sys.path.insert(0, os.path.dirname(HERE))
    import oracle
    n = rows * cols
    q, k, v = oracle.synthetic_qkv(1234, n, (window + 1) * n, d)
    case = oracle.Ref().case(q, k, v, [32], list(range(32 - window, 33)), rows, cols, oracle.Mask.all())
    case.dense_stream(oracle.head_scale(d), 8)
    t = time.perf_counter()
    case.dense_stream(oracle.head_scale(d), sample_rows)
    dt = time.perf_counter() - t
    step_s = dt * (n / sample_rows) * heads
    return {"what": "dense_attention_stream (P/src/attention.cpp:58-99), single thread (the reference has no "
                    "threaded dense path)", "sample": f"{sample_rows} query rows of one head, "
            f"{dt*1e3:.1f} ms, extrapolated x{n / sample_rows:.0f} rows x {heads} heads", "layer_step_s": step_s,
            "query_tokens_per_s": n / step_s}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(os.path.dirname(HERE), "profiles", "r2_configs.json"))
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    res = {"note": "step: CUDA events around the loop; front/attention: per-class spans (second pass); synthetic "
                   "N(0,1) bf16; 4*d FLOP per executed pair", "peak_tflops": PEAK, "peak_source": PEAK_SRC,
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
    try:
        res["cpu_dense_causal"] = cpu_dense_stream()
    except Exception as e:  # oracle/_ref not built on this box
        res["cpu_dense_causal"] = {"unavailable": repr(e)}
    head = res["points"][0]
    res["stack_30x32"] = {"layer_steps": 960, "attention_stack_ms_extrapolated": head["step_us"] * 960 / 1e3,
                          "note": "960 layer-steps x the measured headline layer-step time (append + mask "
                                  "builder + attention, fvsr_ring_step), extrapolated, 1 GPU"}
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
