"""Regenerate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run in the build container (needs /root/reference to compile oracle/_ref):

    python tests/golden/make_golden.py

Each fixture is one seeded case of the reference's own operator pair
(plan_sparse -> sparse_attention_exec, P/include/vsr/sparse.hpp:45-64), computed by
the compiled reference sources through oracle/ref_shim.cpp.  Inputs are NOT stored:
they are re-drawn from vsr::Rng(seed) (mt19937_64 + Box-Muller, P/include/vsr/rng.hpp:
12-53) in the reference draw order (q, k, v; P/src/bench.cpp:78-81), so a fixture pins
the generator too.  Stored: the plan (selected ids, counts, diagonal, coarse scores as
raw fp32 bits, coarse-allowed), the fp32 output, its FNV-1a64 (P/include/vsr/common.hpp:
56-64) and the sparsity report.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402  (test infrastructure)

# name, seed, d, q frames, k frames, rows, cols, mask, topk, bf16 inputs
CASES = [
    # SURVEY 8(c) known answers: tiny config, interpretation A (streaming step: query frame 1
    # over context {0,1}) and B (self-attention over 2x16x16); fp32 inputs, d=64, topk=2.
    ("tiny_A", 2510, 64, [1], [0, 1], 16, 16, ("all",), 2, False),
    ("tiny_B", 2510, 64, [0, 1], [0, 1], 16, 16, ("all",), 2, False),
    # the reference fixture generator's own shape (P/src/bench.cpp:281-283: 512 x 32)
    ("bench_512x32", 1234, 32, [0, 1], [0, 1], 16, 16, ("all",), 2, False),
    # bf16-rounded inputs (what the GPU path consumes), streaming shapes
    ("stream_w2_bf16", 401, 128, [5], [3, 4, 5], 24, 40, ("all",), 5, True),
    ("stream_odd_oldest", 402, 64, [6], [3, 4, 5, 6], 16, 24, ("all",), 3, True),
    ("two_frame_q", 403, 128, [4, 5], [2, 3, 4, 5], 16, 32, ("all",), 4, True),
    ("ragged_20x28", 404, 64, [3], [1, 2, 3], 20, 28, ("all",), 4, True),
    ("locality_trunc", 405, 64, [4], [2, 3, 4], 32, 48, ("loc", 12, 20, True), 4, True),
    ("locality_pres", 405, 64, [4], [2, 3, 4], 32, 48, ("loc", 12, 20, False), 4, True),
    ("locality_full_trunc", 406, 64, [2], [1, 2], 16, 16, ("loc", 16, 16, True), 3, True),
    ("saturated", 407, 64, [3], [1, 2, 3], 16, 24, ("all",), 1000, True),
    ("diag_only", 408, 64, [2], [0, 1, 2], 16, 16, ("all",), 1, True),
    ("causal_bitmask", 409, 64, [0, 1], [0, 1], 16, 16, ("causal",), 2, True),
    ("ties_identical", 0, 32, [1], [0, 1], 16, 16, ("all",), 3, "ties"),
]


def make_mask(spec, lq, lk, case_qf, case_kf, rows, cols):
    if spec[0] == "all":
        return oracle.Mask.all()
    if spec[0] == "loc":
        return oracle.Mask.locality(spec[1], spec[2], truncated=spec[3])
    if spec[0] == "causal":  # token-level causal over the shared token order
        bits = np.zeros((lq, (lk + 63) // 64), np.uint64)
        off = lk - lq
        for i in range(lq):
            n = i + off + 1
            full, rem = divmod(n, 64)
            bits[i, :full] = np.uint64(0xFFFFFFFFFFFFFFFF)
            if rem:
                bits[i, full] = np.uint64((1 << rem) - 1)
        return oracle.Mask.bitmask(bits)
    raise ValueError(spec)


def inputs(seed, d, lq, lk, bf16):
    if bf16 == "ties":  # every token identical: all coarse scores tie
        q = np.ones((lq, d), np.float32) * 0.25
        k = np.ones((lk, d), np.float32) * 0.5
        v = np.tile(np.arange(d, dtype=np.float32) / d, (lk, 1))
        return q, k, v
    return oracle.synthetic_qkv(seed, lq, lk, d, gen=oracle.Port(), bf16=bool(bf16))


def main():
    ref = oracle.Ref()
    index = {}
    for name, seed, d, qf, kf, rows, cols, mspec, topk, bf16 in CASES:
        lq, lk = len(qf) * rows * cols, len(kf) * rows * cols
        q, k, v = inputs(seed, d, lq, lk, bf16)
        mask = make_mask(mspec, lq, lk, qf, kf, rows, cols)
        case = ref.case(q, k, v, qf, kf, rows, cols, mask)
        plan = case.plan(topk)
        scale = oracle.head_scale(d)
        out = case.exec(scale)
        rep = case.report()
        fnv = oracle.fnv1a64(out.tobytes())
        np.savez_compressed(
            os.path.join(HERE, f"{name}.npz"),
            sel=plan.sel, count=plan.count, diag=plan.diag,
            coarse_bits=plan.coarse.view(np.uint32), allowed=plan.allowed,
            out=out, mask_bits=(mask.bits if mask.kind == 2 else np.zeros((0, 0), np.uint64)))
        index[name] = {
            "seed": seed, "d": d, "q_frames": qf, "k_frames": kf, "rows": rows, "cols": cols,
            "mask": list(mspec), "topk": topk, "inputs": ("ties" if bf16 == "ties" else ("bf16" if bf16 else "fp32")),
            "scale": scale, "fnv1a64": f"{fnv:016x}", "density": rep["density"],
            "executed_flops": rep["executed_flops"], "dense_flops": rep["dense_flops"],
            "selected": plan.lists(),
        }
        print(f"{name:22s} bnq={plan.bnq:3d} fnv={fnv:016x} density={rep['density']:.4f}")
    with open(os.path.join(HERE, "index.json"), "w") as f:
        json.dump(index, f, indent=1)


if __name__ == "__main__":
    main()
