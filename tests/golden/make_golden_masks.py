"""Regenerate tests/golden/token_masks.npz from the UNMODIFIED reference (oracle/_ref).

    python tests/golden/make_golden_masks.py

build_segment_mask / build_causal_mask (P/src/mask.cpp:67-101) on seeded labels, stored as
MaskMatrix words (P/include/vsr/mask.hpp:16-59), plus the labels themselves.  Sizes straddle
the 64-bit word boundary (63, 64, 65) and one streaming-sized case (2 frames x 16x24)."""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402  (test infrastructure)


def main():
    ref = oracle.Ref()
    rng = np.random.default_rng(2510)
    arrays = {}
    for L in (1, 63, 64, 65, 300, 768):
        seg = np.unique(rng.integers(0, 6, L), return_inverse=True)[1].astype(np.int32)
        arrays[f"seg{L}.labels"] = seg
        arrays[f"seg{L}.bits"] = ref.segment_mask(seg)
        frame = np.sort(rng.integers(0, 4, L)).astype(np.int32)
        arrays[f"causal{L}.labels"] = frame
        for la in (0, 1):
            arrays[f"causal{L}.la{la}.bits"] = ref.causal_mask(frame, la)
    np.savez_compressed(os.path.join(HERE, "token_masks.npz"), **arrays)
    print("wrote", os.path.join(HERE, "token_masks.npz"))


if __name__ == "__main__":
    main()
