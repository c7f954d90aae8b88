"""Shared helpers for the parity tests (oracle = oracle/ CPU restatement, test-only)."""
from __future__ import annotations

import numpy as np

import oracle

# Output tolerance of the bf16 tensor-core path against the fp32 oracle fed the same
# bf16-rounded inputs: relative L2 and max-abs, per layer shape.
REL_L2_TOL = 5e-3
MAX_ABS_TOL = 2e-2


def qkv(seed: int, heads: int, lq: int, lk: int, d: int, scale_q: float = 1.0):
    """Per-head q, k, v drawn from vsr::Rng(seed + h) in reference order, bf16-rounded."""
    port = oracle.Port()
    qs, ks, vs = [], [], []
    for h in range(heads):
        q, k, v = oracle.synthetic_qkv(seed + h, lq, lk, d, gen=port, bf16=False)
        qs.append(oracle.bf16_round(q * np.float32(scale_q)))
        ks.append(k)
        vs.append(v)
    return (np.stack(qs), oracle.bf16_round(np.stack(ks)), oracle.bf16_round(np.stack(vs)))


def to_dev(x: np.ndarray):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to("cuda").to(torch.bfloat16)


def rel_l2(out: np.ndarray, ref: np.ndarray) -> float:
    den = float(np.linalg.norm(ref.astype(np.float64)))
    return float(np.linalg.norm(out.astype(np.float64) - ref.astype(np.float64))) / max(den, 1e-30)


def max_abs(out: np.ndarray, ref: np.ndarray) -> float:
    return float(np.max(np.abs(out.astype(np.float64) - ref.astype(np.float64)))) if out.size else 0.0


def oracle_plans(q, k, qf, kf, rows, cols, mask, topk):
    port = oracle.Port()
    return [port.plan(q[h], k[h], qf, kf, rows, cols, mask, topk) for h in range(q.shape[0])]


def oracle_outs(q, k, v, qf, kf, rows, cols, mask, plans, scale, row_begin=0, row_end=-1):
    port = oracle.Port()
    return np.stack([port.exec(q[h], k[h], v[h], qf, kf, rows, cols, mask, plans[h], scale, row_begin, row_end)
                     for h in range(q.shape[0])])


def to_oracle_mask(m):
    """paper_2510_12747_b200.Mask -> oracle.Mask (bitmask passes host bits)."""
    from paper_2510_12747_b200 import Mask
    if m is None or m.kind == 0:
        return oracle.Mask.all()
    if m.kind == 1:
        return oracle.Mask.locality(m.extent_h, m.extent_w, truncated=(m.mode == 1))
    return oracle.Mask.bitmask(m.bits.cpu().numpy().view(np.uint64))


def par_map(fn, items, workers=None):
    """Run oracle calls in threads (the C port releases the GIL inside ctypes calls); each
    call must build its own oracle.Port (Port keeps per-instance keep-alive buffers)."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    items = list(items)
    workers = workers or max(1, min(len(items), os.cpu_count() or 1))
    with ThreadPoolExecutor(max_workers=workers) as ex:
        return list(ex.map(fn, items))


def record_parity(case: str, **fields) -> None:
    """Append one per-shape parity line (rel_l2, max_abs, ...) to $FVSR_PARITY_REPORT (JSON
    lines) when set; tools/parity_report.py turns it into profiles/parity_*.json."""
    import json
    import os
    path = os.environ.get("FVSR_PARITY_REPORT")
    if not path:
        return
    with open(path, "a") as f:
        f.write(json.dumps({"case": case, **fields}) + "\n")
