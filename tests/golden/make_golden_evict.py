"""Regenerate tests/golden/evict_mass.npz from the UNMODIFIED reference (oracle/_ref).

Run in the build container (needs /root/reference to compile oracle/_ref):

    python tests/golden/make_golden_evict.py

Scored eviction, computed by the compiled reference through
oracle/ref_shim.cpp:
  * frame_attention_mass(plan, key_grid) (P/src/kv_cache.cpp:170-206) for seeded plans
    (bf16-rounded vsr::Rng inputs, so the GPU plan sees identical values), including a
    non-contiguous key frame set (what uniform eviction leaves behind) and a locality mask;
  * KVCache::evict (P/src/kv_cache.cpp:97-137) for the three strategies on seeded scores,
    with exact ties (older frame goes first).
Stored: case metadata (JSON), the coarse scores / allowed bits of each plan, the reference
masses (float64) and the retained frame ids per head.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402  (test infrastructure)

# name, seed, d, q frames, k frames, rows, cols, mask, topk
MASS_CASES = [
    ("w4_all", 501, 128, [6], [2, 3, 4, 5, 6], 24, 40, ("all",), 5),
    ("gap_all", 502, 64, [7], [2, 4, 6, 7], 16, 24, ("all",), 4),
    ("loc_trunc", 503, 64, [5], [2, 3, 4, 5], 20, 28, ("loc", 9, 9, True), 3),
    ("two_frame_q", 504, 128, [4, 5], [1, 3, 4, 5], 16, 32, ("all",), 4),
]
# name, seed, strategy, window, ids, heads, tie
EVICT_CASES = [
    ("sliding", 601, 0, 3, [3, 4, 5, 6, 7], 2, False),
    ("uniform", 602, 1, 3, [3, 4, 5, 6, 7], 3, False),
    ("uniform_ties", 603, 1, 2, [1, 2, 4, 5, 8], 2, True),
    ("headwise", 604, 2, 2, [0, 1, 2, 3, 4, 5], 3, False),
    ("uniform_under", 605, 1, 6, [3, 4, 5], 2, False),
]


def mask_of(spec):
    if spec[0] == "all":
        return oracle.Mask.all()
    return oracle.Mask.locality(spec[1], spec[2], spec[3])


def main():
    ref = oracle.Ref()
    arrays, meta = {}, {"mass": [], "evict": []}
    for name, seed, d, qf, kf, rows, cols, mspec, topk in MASS_CASES:
        n = rows * cols
        q, k, v = oracle.synthetic_qkv(seed, len(qf) * n, len(kf) * n, d)
        c = ref.case(q, k, v, qf, kf, rows, cols, mask_of(mspec))
        plan = c.plan(topk)
        arrays[f"{name}.coarse"] = plan.coarse
        arrays[f"{name}.allowed"] = plan.allowed
        arrays[f"{name}.sel"] = plan.sel
        arrays[f"{name}.mass"] = c.frame_mass()
        meta["mass"].append(dict(name=name, seed=seed, d=d, qf=qf, kf=kf, rows=rows, cols=cols, mask=list(mspec),
                                 topk=topk))
    for name, seed, strategy, window, ids, heads, tie in EVICT_CASES:
        rng = np.random.default_rng(seed)
        sc = rng.random((heads, len(ids)))
        if tie:
            sc[:] = np.round(sc * 2) / 2  # exact ties across frames
        arrays[f"{name}.scores"] = sc
        kept = ref.kv_evict(strategy, window, ids, sc, heads)
        arrays[f"{name}.kept"] = np.array(kept, np.int32) if len({len(x) for x in kept}) == 1 else np.array(
            [x + [-1] * (len(ids) - len(x)) for x in kept], np.int32)
        meta["evict"].append(dict(name=name, strategy=strategy, window=window, ids=ids, heads=heads))
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), np.uint8)
    np.savez_compressed(os.path.join(HERE, "evict_mass.npz"), **arrays)
    print("wrote", os.path.join(HERE, "evict_mass.npz"))


if __name__ == "__main__":
    main()
