"""GPU token-mask builders (build_segment_mask / build_causal_mask, P/src/mask.cpp:67-101):
device MaskMatrix words bit-exact with the reference fixtures, the reference's error
behaviour, and the built mask driving plan + attention through the bitmask path."""
import os

import numpy as np
import pytest
import torch

import oracle
from tests.helpers import MAX_ABS_TOL, REL_L2_TOL, max_abs, oracle_outs, oracle_plans, rel_l2, to_dev

pytestmark = pytest.mark.gpu
fv = pytest.importorskip("paper_2510_12747_b200")
MASKS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "token_masks.npz")


def _words(mask):
    return mask.bits.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("L", (1, 63, 64, 65, 300, 768))
def test_token_masks_bit_exact(L):
    z = np.load(MASKS)
    assert np.array_equal(_words(fv.build_segment_mask(z[f"seg{L}.labels"])), z[f"seg{L}.bits"])
    for la in (0, 1):
        got = _words(fv.build_causal_mask(z[f"causal{L}.labels"], la))
        assert np.array_equal(got, z[f"causal{L}.la{la}.bits"])


def test_large_masks_match_oracle():  # 2 frames of 768x1408 latent (8448 tokens), random labels
    rng = np.random.default_rng(5)
    L = 2 * 48 * 88
    seg = rng.permutation(np.arange(L) % 7).astype(np.int32)
    assert np.array_equal(_words(fv.build_segment_mask(seg)), oracle.segment_mask(seg))
    frame = np.repeat(np.arange(2), L // 2).astype(np.int32)
    assert np.array_equal(_words(fv.build_causal_mask(frame, 0)), oracle.causal_mask(frame, 0))


def test_token_mask_errors():
    with pytest.raises(fv.ConfigError):
        fv.build_segment_mask([0, 2])
    with pytest.raises(fv.ConfigError):
        fv.build_segment_mask([-1, 0])
    with pytest.raises(fv.ConfigError):
        fv.build_causal_mask([1, 0], 0)
    with pytest.raises(fv.ConfigError):
        fv.build_causal_mask([0, 1], -1)


@pytest.mark.parametrize("kind", ["segment", "causal"])
def test_built_mask_drives_plan_and_attention(kind):
    """Self-attention over 2 frames (plan_sparse self form, as bench_sparsity runs it) with a
    device-built stage-1 segment mask (Eq. 1) or a frame-causal mask."""
    heads, rows, cols, d, topk, qf = 2, 16, 24, 64, 3, [0, 1]
    n = rows * cols
    L = 2 * n
    if kind == "segment":  # two segments: the top and bottom half of every frame
        lab = np.tile(np.repeat([0, 1], n // 2), 2).astype(np.int32)
        fmask, bits = fv.build_segment_mask(lab), oracle.segment_mask(lab)
    else:
        lab = np.repeat([0, 1], n).astype(np.int32)
        fmask, bits = fv.build_causal_mask(lab, 0), oracle.causal_mask(lab, 0)
    omask = oracle.Mask.bitmask(bits)
    port = oracle.Port()
    x = oracle.bf16_round(np.stack([port.gaussian(900 + h, 3 * L * d).reshape(3, L, d) for h in range(heads)]))
    q, k, v = x[:, 0], x[:, 1], x[:, 2]
    g = fv.TokenGrid(qf, rows, cols)
    plan = fv.plan_sparse(to_dev(q), to_dev(k), g, g, fmask, topk)
    out = fv.sparse_attention_exec(to_dev(q), to_dev(k), to_dev(v), plan, fmask).float().cpu().numpy()
    refs = oracle_plans(q, k, qf, qf, rows, cols, omask, topk)
    ref = oracle_outs(q, k, v, qf, qf, rows, cols, omask, refs, oracle.head_scale(d))
    for h in range(heads):
        assert plan.selected(h) == refs[h].lists()
    assert rel_l2(out, ref) <= REL_L2_TOL and max_abs(out, ref) <= MAX_ABS_TOL
