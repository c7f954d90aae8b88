#!/usr/bin/env python
"""Benchmark: FlashVSR block-sparse streaming attention layer-step on B200.

Metric (BASELINE.json): sparse-attn tokens/s & effective TFLOP/s at the 768x1408 latent
(48x88 tokens/frame), 12 heads, d=128, sliding window W=4 (context = 5 frames), top-k 27
(= topk_for_density(0.136, 198), P/src/bench.cpp:62-69), all-allowed token mask.

One step = one streaming layer-step of the hot path for every head: append the new
frame's K/V to the device ring (KVCache::append), build the plan (pool Q, score against the
ring's pooled K partials, top-k with forced diagonal), block-sparse attention over the
ring, sliding evict.  Steps cycle over a 30-layer stack of rings (BASELINE config #3), so
each step's inputs (127 MB of ring per layer, 3.8 GB total) are larger than L2.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

N>1 runs under torchrun: (head, q-tile) units are sharded across ranks (head parallel),
outputs gathered with NCCL all_gather_into_tensor on NCCL's stream, overlapped with the
next layer-step; time is the max over ranks.  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

ROWS, COLS, HEADS, D, WINDOW, TOPK, LAYERS = 48, 88, 12, 128, 4, 27, 30
T0 = 32  # steady state: query frame t=32 over context {28..32}
POOL = 4  # distinct synthetic frames cycled through the stream
METRIC = "sparse-attn tokens/s & effective TFLOP/s at 768×1408 latent, 1/2/4/8 B200 vs CPU"
WORKLOAD = ("768x1408 streaming layer-step: 48x88 latent tokens/frame, 12 heads, d=128, KV window W=4 "
            "(context 5 frames, 198 key blocks), top-k 27 (13.6%), all-allowed mask, Tq=1")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return {"hbm_gbs": p["hbm_gbs"], "bf16_tflops": p["bf16_tflops"],
                "bf16_tflops_sustained": p.get("bf16_tflops_sustained"), "source": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


# ------------------------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ------------------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None
        self.window = (0.0, 0.0)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), line.strip()))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        t0, t1 = self.window
        rows = [s for (t, s) in self.samples if t0 - 0.05 <= t <= t1 + 0.05] or [s for (_, s) in self.samples]
        mhz, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            parts = [x.strip() for x in r.split(",")]
            if len(parts) < 6:
                continue
            try:
                mhz.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(mhz) if mhz else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(mhz)}


# ------------------------------------------------------------------------------------------
# CPU baseline: the reference hot path (oracle/_ref, compiled from /root/reference) on host cores
# ------------------------------------------------------------------------------------------
def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def reference_cases():
    """The 12 heads of the step at t=32 over {28..32}: per-head q/k/v drawn from
    vsr::Rng(1234 + head) (fp32 values that are bf16-representable), as compiled-reference
    cases (oracle/_ref; None when it is not built)."""
    import oracle
    N = ROWS * COLS
    try:
        ref = oracle.Ref()
    except Exception:
        return None
    cases = []
    for h in range(HEADS):
        q, k, v = oracle.synthetic_qkv(1234 + h, N, 5 * N, D)
        cases.append(ref.case(q, k, v, [T0], list(range(T0 - WINDOW, T0 + 1)), ROWS, COLS, oracle.Mask.all()))
    return cases


def time_reference_steps(n_steps: int, threads: int, warmup: int = 1):
    """Wall seconds of whole layer-steps of the reference hot path: head_attention (partition,
    mask, plan_sparse, sparse_attention_exec; P/src/stream.cpp:175-194) for each of the 12
    heads, distinct per-head inputs, `threads` worker threads per call.  Plus one head at
    threads=1 (reported separately, x12 extrapolated and labelled so)."""
    import oracle
    scale = oracle.head_scale(D)
    cases = reference_cases()
    if cases is None:  # no compiled reference: the C port, one head per step, x12
        port = oracle.Port()
        q, k, v = oracle.synthetic_qkv(1234, ROWS * COLS, 5 * ROWS * COLS, D)
        kf = list(range(T0 - WINDOW, T0 + 1))
        times = []
        for i in range(warmup + n_steps):
            t = time.perf_counter()
            plan = port.plan(q, k, [T0], kf, ROWS, COLS, oracle.Mask.all(), TOPK)
            port.exec(q, k, v, [T0], kf, ROWS, COLS, oracle.Mask.all(), plan, scale)
            if i >= warmup:
                times.append((time.perf_counter() - t) * HEADS)
        return statistics.median(times), "port", 1, times, None
    times = []
    for i in range(warmup + n_steps):
        t = time.perf_counter()
        for c in cases:
            c.head_attention(TOPK, scale, threads)
        if i >= warmup:
            times.append(time.perf_counter() - t)
    t = time.perf_counter()
    cases[0].head_attention(TOPK, scale, 1)
    t1_head = time.perf_counter() - t
    return statistics.median(times), "reference", threads, times, t1_head


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = cpu_threads()
    # each step = one whole 12-head layer-step of the reference; at most 8 timed steps (+1
    # warm-up) so the arm ends within a couple of minutes for any --steps
    n_timed = max(1, min(args.steps, 8))
    med, kind, threads_used, times, t1_head = time_reference_steps(n_timed, threads, warmup=1)
    tokens_per_s = ROWS * COLS / med
    sample = (f"{n_timed} whole layer-steps (12 head_attention calls each, distinct per-head inputs), median "
              f"{med*1e3:.1f} ms/step, threads={threads_used}, {cpu_model()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": tokens_per_s, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": n_timed, "steps_requested": args.steps, "warmup": 1, "ms_per_step": med * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (vsr::Rng N(0,1), bf16-representable), per-head seeds 1234+h",
        "config": {"workload": WORKLOAD, "heads": HEADS, "d": D, "latent": [ROWS, COLS], "window": WINDOW,
                   "topk": TOPK, "mask": "all"},
        "cpu_baseline": {"value": tokens_per_s, "unit": "tokens/s", "cores": threads_used, "kind": kind,
                         "sample": sample},
        "e2e": {"value": tokens_per_s, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if t1_head is not None:
        line["cpu_threads1"] = {"value": ROWS * COLS / (t1_head * HEADS), "unit": "tokens/s", "cores": 1,
                                "sample": f"one head_attention call at threads=1 ({t1_head*1e3:.0f} ms), x12 heads "
                                          "(extrapolated)"}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------
# B200 arm
# ------------------------------------------------------------------------------------------
def run_b200(args):
    import torch
    import torch.distributed as dist
    import paper_2510_12747_b200 as fv
    from paper_2510_12747_b200 import _abi, head_parallel as hp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    N = ROWS * COLS
    tiles = ((ROWS + 7) // 8) * ((COLS + 7) // 8)
    units = HEADS * tiles
    sh = hp.shard(units, tiles, world, rank)
    nh = sh.heads
    ctx = fv.Context.default()
    mask = fv.Mask.all_allowed()
    scale = 1.0 / math.sqrt(D)

    # synthetic pool: POOL frames of q/k/v, N(0,1) rounded to bf16, generated on device
    gen = torch.Generator(device=dev).manual_seed(2510)
    pool = [[torch.randn((HEADS, N, D), generator=gen, device=dev).to(torch.bfloat16) for _ in range(3)]
            for _ in range(POOL)]
    pool_local = [[x[sh.h0:sh.h1].contiguous() for x in fr] for fr in pool]

    rings = fv.KVRing(LAYERS, nh, D, ROWS, COLS, WINDOW, ctx=ctx)
    for l in range(LAYERS):
        for f in range(T0 - WINDOW, T0):
            _, k, v = pool_local[(f + l) % POOL]
            rings.append(l, f, k, v)
            rings.evict(l)
    torch.cuda.synchronize()

    gather = hp.Gatherer(sh, D, dev) if world > 1 else None
    out_tok = torch.empty((HEADS, N, D), dtype=torch.bfloat16, device=dev)
    lib = ctx.lib
    md = mask.c()
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    import ctypes as C

    state = {"s": 0}

    def step(md=md):
        s = state["s"]
        state["s"] += 1
        l = s % LAYERS
        t = T0 + s // LAYERS
        q, k, v = pool_local[(t + l) % POOL]
        ids = (C.c_int32 * 1)(t)
        # one C-ABI call: ring append + mask builder (one launch) + sparse attention
        if gather is None:
            _abi.check(lib.fvsr_ring_step(ctx.h, rings.h, l, t, k.data_ptr(), v.data_ptr(), q.data_ptr(), ids, 1,
                                          C.byref(md), TOPK, scale, 0, -1, out_tok.data_ptr(), 0, 0, None, None,
                                          C.c_void_p(sptr)))
        else:
            buf = gather.next_shard()
            _abi.check(lib.fvsr_ring_step(ctx.h, rings.h, l, t, k.data_ptr(), v.data_ptr(), q.data_ptr(), ids, 1,
                                          C.byref(md), TOPK, scale, sh.local_unit_begin, sh.local_unit_end,
                                          buf.data_ptr(), 1, 0, None, None, C.c_void_p(sptr)))
            gather.launch()
        _abi.check(lib.fvsr_ring_evict_sliding(rings.h, l))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- warmup ---------------------------------------------------------------------------
    for _ in range(args.warmup):
        step()
    if gather:
        gather.drain()
    ctx.check_errors()
    ctx.read_pairs()  # reset the executed-pair counter
    ctx.timing_read(_abi.TIME_ATTENTION, clear=True)

    # ---- timed region -----------------------------------------------------------------------
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    launches0 = ctx.launch_count()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.time()
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    w_enq = time.time()
    if gather:
        gather.drain()
    ev1.record(stream)
    barrier()
    w1 = time.time()
    clocks.window = (w0, w1)
    time.sleep(0.15)
    clocks.stop()
    elapsed_ms = ev0.elapsed_time(ev1)
    launches = ctx.launch_count() - launches0
    ctx.check_errors()
    pairs = ctx.read_pairs()
    # per-kernel-class CUDA-event spans, in a separate pass after the timed region (events
    # between the kernels would serialise their programmatic-dependent-launch overlap)
    span_steps = min(args.steps, 200)
    ctx.read_tiles()  # reset the key-tile counters
    ctx.timing(True)
    for _ in range(span_steps):
        step()
    if gather:
        gather.drain()
    barrier()
    ctx.timing(False)
    ctx.check_errors()
    pairs_span = ctx.read_pairs()
    tiles_span, full_span = ctx.read_tiles()
    attn_ms, attn_n = ctx.timing_read(_abi.TIME_ATTENTION)
    pk_ms, pk_n = ctx.timing_read(_abi.TIME_PACK)
    se_ms, se_n = ctx.timing_read(_abi.TIME_SELECT)
    fr_ms, fr_n = ctx.timing_read(_abi.TIME_FRONT, clear=True)
    # the same step with the paper's locality window at 768x1408 (48x72 latent tokens, truncated;
    # SURVEY 8(d)), measured the same way (spans + kernel-counted pairs)
    variants = {}
    if world == 1:
        mloc = fv.Mask.locality(48, 72, truncated=True).c()
        for _ in range(10):
            step(mloc)
        barrier()
        ctx.read_pairs()
        ctx.timing(True)
        ev_a, ev_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev_a.record(stream)
        nv = min(args.steps, 100)
        for _ in range(nv):
            step(mloc)
        ev_b.record(stream)
        barrier()
        ctx.timing(False)
        ctx.check_errors()
        vp = ctx.read_pairs()
        va_ms, va_n = ctx.timing_read(_abi.TIME_ATTENTION)
        ctx.timing_read(_abi.TIME_FRONT, clear=True)
        v_step = ev_a.elapsed_time(ev_b) / nv  # includes the span events (serialises the PDL overlap)
        v_attn = va_ms / max(1, va_n)
        v_eff = 4.0 * D * vp / max(1, va_n) / (v_attn / 1e3) / 1e12
        variants["locality_48x72_truncated"] = {
            "mask": "locality 48x72 truncated", "attention_us": v_attn * 1e3, "eff_tflops": v_eff,
            "frac": v_eff / peaks()["bf16_tflops"], "executed_pairs_per_launch": vp / max(1, va_n),
            "step_us_with_span_events": v_step * 1e3, "tokens_per_s_with_span_events": N / (v_step / 1e3)}
    if world > 1:
        t = torch.tensor([elapsed_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
        pt = torch.tensor([float(pairs), attn_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(pt, op=dist.ReduceOp.SUM)
        pairs_total = int(pt[0].item())
    else:
        pairs_total = pairs

    ms_per_step = elapsed_ms / args.steps
    tokens_per_s = N * args.steps / (elapsed_ms / 1e3)
    eff_tflops = 4.0 * D * pairs_total / (elapsed_ms / 1e3) / 1e12
    pk = peaks()

    # ---- end-to-end through the C-ABI with host buffers -------------------------------------
    e2e = None
    h2d = 3 * nh * N * D * 2
    d2h = (HEADS if world == 1 else HEADS) * N * D * 2
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    hq = [[x.cpu().pin_memory() for x in fr] for fr in pool_local]
    # Streaming pipeline: consecutive layer-steps (different layers, independent rings) go to
    # alternating (context, stream) pairs, so step s+1's H2D copy overlaps step s's kernels
    # and step s-1's D2H read.  Every step still copies its own inputs in and its output out.
    n_pipe = 2 if world == 1 else 1
    ctxs = [ctx] + [fv.Context() for _ in range(n_pipe - 1)]
    streams = [stream] + [torch.cuda.Stream(device=dev) for _ in range(n_pipe - 1)]
    hos = [torch.empty((HEADS, N, D), dtype=torch.bfloat16).pin_memory() for _ in range(n_pipe)]
    ho = hos[0]
    if world == 1:  # size each context's staging buffers outside the timed region
        for j in range(n_pipe):
            s = state["s"]
            state["s"] += 1
            l, t = s % LAYERS, T0 + s // LAYERS
            q, k, v = hq[(t + l) % POOL]
            _abi.check(lib.fvsr_ring_step_host(ctxs[j].h, rings.h, l, t, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                               C.byref(md), TOPK, scale, hos[j].data_ptr(),
                                               C.c_void_p(streams[j].cuda_stream)))
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for st in streams[1:]:
        st.wait_event(e0)
    for i in range(e2e_steps):
        s = state["s"]
        state["s"] += 1
        l = s % LAYERS
        t = T0 + s // LAYERS
        q, k, v = hq[(t + l) % POOL]
        if world == 1:
            j = i % n_pipe
            _abi.check(lib.fvsr_ring_step_host(ctxs[j].h, rings.h, l, t, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                               C.byref(md), TOPK, scale, hos[j].data_ptr(),
                                               C.c_void_p(streams[j].cuda_stream)))
        else:
            qd, kd, vd = (x.to(dev, non_blocking=True) for x in (q, k, v))
            buf = gather.next_shard()
            rings.step(l, t, kd, vd, qd, [t], mask, TOPK, unit_begin=sh.local_unit_begin, unit_end=sh.local_unit_end,
                       out=buf[: sh.u1 - sh.u0], tile_major=True, check_errors=False)
            gather.launch()
            full = gather.result()
            ho.view(-1)[: full.numel()].copy_(full.reshape(-1)[: ho.numel()], non_blocking=True)
            rings.evict(l)
    for st in streams[1:]:
        ev = torch.cuda.Event()
        ev.record(st)
        stream.wait_event(ev)
    e1.record(stream)
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    for c_, st in zip(ctxs, streams):
        c_.check_errors(st)
    e2e = {"value": N * e2e_steps / (e2e_ms / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "steps": e2e_steps, "ms_per_step": e2e_ms / e2e_steps,
           "path": f"fvsr_ring_step_host (C-ABI, pinned host buffers), {n_pipe} contexts/streams pipelined"
                   if world == 1 else
                   "python composition over the C-ABI + NCCL gather, pinned host buffers"}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel ---------------------------------------------------
    attn_avg_ms = attn_ms / max(1, attn_n)
    pairs_per_launch = pairs_span / max(1, attn_n)
    achieved = 4.0 * D * pairs_per_launch / (attn_avg_ms / 1e3) / 1e12
    traffic, traffic_src = None, None
    prof = os.path.join(HERE, "profiles", "ncu_attention_r2.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                pj = json.load(f)
            traffic = pj.get("dram_bytes_per_launch")
            traffic_src = ("ncu --set full of this kernel at this workload (not measured in this run): "
                           f"profiles/ncu_attention_r2.json, {pj.get('source', '')}")
        except Exception:
            traffic = None
    roofline = {"kernel": "sparse_attn_kernel<128>", "bound": "tensor", "achieved": achieved,
                "peak": pk["bf16_tflops"], "unit": "TFLOP/s", "frac": achieved / pk["bf16_tflops"],
                "frac_sustained": achieved / pk["bf16_tflops_sustained"] if pk["bf16_tflops_sustained"] else None,
                "peak_source": pk["source"] + " burst bf16 (MEASURED_PEAKS.json)", "traffic": traffic,
                "traffic_source": traffic_src,
                "flops_per_launch": 4.0 * D * pairs_per_launch,
                "flop_def": "4*d per executed (mask-allowed, selected-block) token pair, counted by the kernel",
                "avg_launch_us": attn_avg_ms * 1e3, "launches": attn_n}
    # tile-level tensor work (every issued MMA, incl. masked/padding lanes): QK^T over 128 key
    # rows and PV over the tile's valid rows (128, or 64 for a lone single-frame block)
    nt_l, nf_l = tiles_span / max(1, attn_n), full_span / max(1, attn_n)
    tile_flops = nt_l * 2 * 128 * 64 * D + (nf_l * 128 + (nt_l - nf_l) * 64) * 2 * 64 * D
    roofline["tiles_per_launch"] = nt_l
    roofline["full_tiles_per_launch"] = nf_l
    roofline["tile_tflops"] = tile_flops / (attn_avg_ms / 1e3) / 1e12
    roofline["tile_flops_per_launch"] = tile_flops
    # the K/V gather (L2 -> shared memory, cp.async.bulk): the attention kernel's binding
    # resource: bytes each launch moves into shared memory per key tile
    # (16 KB frame-tile halves of K and V) plus each unit's Q tile, against the measured
    # per-SM bulk-copy ingest cap (tools/l2bench, profiles/l2bench_r2.json)
    tile_b = 128 * D
    gather_bytes = (nf_l * 2 + (nt_l - nf_l)) * tile_b * 2 + HEADS * tiles * tile_b
    l2cap = None
    try:
        with open(os.path.join(HERE, "profiles", "l2bench_r2.json")) as f:
            rows = json.load(f)["rows"]
        l2cap = max(r["GBps"] for r in rows if r["buffer_mb"] == 64 and r["grid"] == 148)
    except Exception:
        pass
    roofline["gather"] = {"bytes_per_launch": gather_bytes, "achieved_gbs": gather_bytes / (attn_avg_ms / 1e3) / 1e9,
                          "peak_gbs": l2cap, "frac": (gather_bytes / (attn_avg_ms / 1e3) / 1e9 / l2cap) if l2cap else None,
                          "peak_source": "L2->SMEM cp.async.bulk ingest, 148 CTAs x 32 KB stages, L2-resident 64 MB "
                                         "(tools/l2bench.cu, profiles/l2bench_r2.json)"}
    fr_avg = fr_ms / max(1, fr_n)
    bnk = 3 * tiles  # context {28..32}: t_rows 14, 15, 16
    # front kernel (ring append + mask builder, one launch): K/V read + written once, their
    # pooled partials written, Q read once and its packed tiles written, the ring's pooled
    # keys read, indices written
    ap_bytes = 2 * 2 * nh * N * D * 2 + nh * tiles * D * 4 * 2
    mb_bytes = nh * N * D * 2 * 2 + nh * bnk * D * 4 + nh * tiles * TOPK * 4
    front = {"kernel": "ring_pack_kernel (append K, V + Q pack/pool) + mask_select_kernel (coarse scores + top-k)", "avg_us": fr_avg * 1e3,
             "algorithmic_bytes": ap_bytes + mb_bytes,
             "gbs": (ap_bytes + mb_bytes) / (fr_avg / 1e3) / 1e9 if fr_avg > 0 else None, "peak_gbs": pk["hbm_gbs"],
             "frac": (ap_bytes + mb_bytes) / (fr_avg / 1e3) / 1e9 / pk["hbm_gbs"] if fr_avg > 0 else None}
    # per launch: the append + query pack is an HBM copy (bound: HBM); the selector reads only
    # the pooled rows and is latency-bound (its bytes are reported, not a bound)
    pack_bytes = 2 * 2 * nh * N * D * 2 + 2 * nh * N * D * 2 + nh * tiles * D * 4 * 5
    sel_bytes = nh * bnk * D * 4 + nh * tiles * D * 4 + nh * tiles * TOPK * 4
    for name, ms, n, nbytes in (("ring_pack", pk_ms, pk_n, pack_bytes), ("mask_select", se_ms, se_n, sel_bytes)):
        avg = ms / max(1, n)
        front[name] = {"avg_us": avg * 1e3, "algorithmic_bytes": nbytes,
                       "gbs": nbytes / (avg / 1e3) / 1e9 if avg > 0 else None,
                       "frac_of_hbm": nbytes / (avg / 1e3) / 1e9 / pk["hbm_gbs"] if avg > 0 else None}

    # ---- CPU baseline (reference on host cores, rank 0, N=1 only) ----------------------------
    cpu = None
    if world == 1 and not args.no_cpu:
        threads = cpu_threads()
        med, kind, threads_used, times, t1_head = time_reference_steps(args.cpu_steps, threads, warmup=0)
        cpu = {"value": N / med, "unit": "tokens/s", "cores": threads_used, "kind": kind,
               "sample": f"{args.cpu_steps} whole layer-steps of the reference (12 head_attention calls each: "
                         f"partition, mask, plan_sparse, sparse_attention_exec), median {med*1e3:.1f} ms/step, "
                         f"threads={threads_used}, {cpu_model()}"}
        if t1_head is not None:
            cpu["threads1"] = {"value": N / (t1_head * HEADS), "unit": "tokens/s", "cores": 1,
                               "sample": f"one head at threads=1 ({t1_head*1e3:.0f} ms), x12 heads (extrapolated)"}

    line = {
        "metric": METRIC, "value": tokens_per_s, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic N(0,1) bf16 (torch.Generator seed 2510, 4-frame pool)",
        "config": {"workload": WORKLOAD, "heads": HEADS, "d": D, "latent": [ROWS, COLS], "window": WINDOW,
                   "topk": TOPK, "mask": "all", "layers_cycled": LAYERS,
                   "l2": "inputs larger than L2: steps cycle 30 layer rings (127 MB each, 3.8 GB)",
                   "parallelism": f"head-parallel x{world}" if world > 1 else "single GPU"},
        "eff_tflops": eff_tflops,
        "roofline": roofline,
        "front": front,
        "variants": variants,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "clocks": clocks.summary(),
        "gpu_launches": launches,
        "host_enqueue_us_per_step": (w_enq - w0) * 1e6 / args.steps,
        "executed_pairs_per_step": pairs_total / args.steps,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=600)
    ap.add_argument("--warmup", type=int, default=30)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=120)
    ap.add_argument("--cpu-steps", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
