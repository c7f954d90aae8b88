"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle.

Plan (mask builder): block indices, counts, diagonal, coarse-allowed bit-exact; coarse
scores bitwise equal.  Exec: bf16 output within REL_L2_TOL / MAX_ABS_TOL of the fp32
oracle fed identical bf16-rounded inputs.  Cases follow the reference's own tests
(P/tests/test_sparse.cpp, test_masks.cpp) plus the BASELINE configs.
"""
import numpy as np
import pytest

import oracle
from tests.helpers import (MAX_ABS_TOL, REL_L2_TOL, max_abs, oracle_outs, oracle_plans, qkv, record_parity, rel_l2,
                           to_dev, to_oracle_mask)

pytestmark = pytest.mark.gpu

fv = pytest.importorskip("paper_2510_12747_b200")


def M(kind="all", eh=1, ew=1, trunc=True):
    if kind == "all":
        return fv.Mask.all_allowed()
    return fv.Mask.locality(eh, ew, truncated=trunc)


# name, seed, heads, q frames, k frames, rows, cols, d, topk, mask
CASES = [
    ("tiny_A_stream_step", 2510, 1, [1], [0, 1], 16, 16, 64, 2, M()),
    ("tiny_B_self", 2510, 1, [0, 1], [0, 1], 16, 16, 64, 2, M()),
    ("ragged_locality_truncated", 1, 3, [5], [2, 3, 4, 5], 20, 28, 64, 3, M("loc", 7, 9, True)),
    ("ragged_locality_preserved", 2, 2, [5], [2, 3, 4, 5], 20, 28, 128, 3, M("loc", 7, 9, False)),
    ("two_latent_chunk_locality", 4, 2, [6, 7], [3, 4, 5, 6, 7], 18, 30, 128, 4, M("loc", 10, 12, True)),
    ("odd_oldest_frame", 9, 2, [33], [29, 30, 31, 32, 33], 24, 40, 128, 5, M()),
    ("scored_eviction_gaps", 11, 2, [40], [31, 34, 35, 38, 40], 16, 24, 64, 3, M()),
    ("saturated_topk", 3, 1, [4, 5], [0, 1, 2, 3, 4, 5], 16, 16, 64, 1000, M()),
    ("full_extent_locality", 5, 1, [2], [0, 1, 2], 12, 20, 64, 4, M("loc", 12, 20, True)),
]


def _gpu_plan(q, k, c):
    name, seed, heads, qf, kf, rows, cols, d, topk, mask = c
    gq, gk = fv.TokenGrid(qf, rows, cols), fv.TokenGrid(kf, rows, cols)
    return fv.plan_sparse(to_dev(q), to_dev(k), gq, gk, mask, topk)


def _assert_plan_equal(plan, refs):
    sel, cnt, diag = plan.sel.cpu().numpy(), plan.count.cpu().numpy(), plan.diagonal_block.cpu().numpy()
    coarse, allowed = plan.coarse_scores.cpu().numpy(), plan.coarse_allowed.cpu().numpy()
    for h, r in enumerate(refs):
        assert sel.shape[1:] == r.sel.shape, (sel.shape, r.sel.shape)
        np.testing.assert_array_equal(cnt[h], r.count)
        np.testing.assert_array_equal(sel[h], r.sel)
        np.testing.assert_array_equal(diag[h], r.diag)
        np.testing.assert_array_equal(allowed[h], r.allowed)
        np.testing.assert_array_equal(coarse[h].view(np.uint32), r.coarse.view(np.uint32))


@pytest.mark.parametrize("c", CASES, ids=[c[0] for c in CASES])
def test_plan_bit_exact(c):
    name, seed, heads, qf, kf, rows, cols, d, topk, mask = c
    q, k, v = qkv(seed, heads, len(qf) * rows * cols, len(kf) * rows * cols, d)
    plan = _gpu_plan(q, k, c)
    refs = oracle_plans(q, k, qf, kf, rows, cols, to_oracle_mask(mask), topk)
    _assert_plan_equal(plan, refs)


@pytest.mark.parametrize("c", CASES, ids=[c[0] for c in CASES])
def test_exec_within_tolerance(c):
    name, seed, heads, qf, kf, rows, cols, d, topk, mask = c
    q, k, v = qkv(seed, heads, len(qf) * rows * cols, len(kf) * rows * cols, d)
    plan = _gpu_plan(q, k, c)
    refs = oracle_plans(q, k, qf, kf, rows, cols, to_oracle_mask(mask), topk)
    scale = oracle.head_scale(d)
    out = fv.sparse_attention_exec(to_dev(q), to_dev(k), to_dev(v), plan, mask, scale).float().cpu().numpy()
    ref = oracle_outs(q, k, v, qf, kf, rows, cols, to_oracle_mask(mask), refs, scale)
    record_parity(name, rows=rows, cols=cols, heads=heads, d=d, topk=topk, q_frames=qf, k_frames=kf,
                  indices_bit_exact=True, rel_l2=rel_l2(out, ref), max_abs=max_abs(out, ref))
    assert rel_l2(out, ref) <= REL_L2_TOL, (name, rel_l2(out, ref))
    assert max_abs(out, ref) <= MAX_ABS_TOL, (name, max_abs(out, ref))


def test_plan_small_head_dims_and_ties():
    """Exact-tie rule and forced diagonal (P/tests/test_sparse.cpp:125-158) at d in {4, 8, 16, 32}."""
    rows = cols = 16
    frames = [0, 1, 2, 3]
    L = 4 * rows * cols
    gq = fv.TokenGrid(frames, rows, cols)
    # identical rows everywhere: every coarse score ties -> lowest ids after the diagonal
    q = np.full((1, L, 4), 0.5, np.float32)
    plan = fv.plan_sparse(to_dev(q), to_dev(q), gq, gq, fv.Mask.all_allowed(), 3)
    for qb, s in enumerate(plan.selected(0)):
        want = sorted({qb} | set([b for b in range(8) if b != qb][:2]))
        assert s == want
    # block 0 keys anti-aligned with every query: block 0 selected only by its own diagonal
    assign, _ = oracle.Port().partition(frames, rows, cols)
    k = np.where(assign[:, None] == 0, -1.0, 1.0).astype(np.float32) * np.ones((1, L, 4), np.float32)
    qq = np.ones((1, L, 4), np.float32)
    plan = fv.plan_sparse(to_dev(qq), to_dev(k), gq, gq, fv.Mask.all_allowed(), 2)
    sel = plan.selected(0)
    assert 0 in sel[0]
    assert all(0 not in s for s in sel[1:])
    for d in (8, 16, 32):
        qn, kn, _ = qkv(77 + d, 2, L, L, d)
        plan = fv.plan_sparse(to_dev(qn), to_dev(kn), gq, gq, fv.Mask.all_allowed(), 2)
        _assert_plan_equal(plan, oracle_plans(qn, kn, frames, frames, rows, cols, oracle.Mask.all(), 2))


def test_bitmask_causal_self_attention():
    """Explicit MaskMatrix path with a causal mask (P/src/mask.cpp:87-102)."""
    import torch
    rows = cols = 16
    frames = [0, 1, 2, 3]
    L = 4 * rows * cols
    fr = np.repeat(np.arange(4), rows * cols)
    allowed = fr[None, :] <= fr[:, None]
    wpr = (L + 63) // 64
    bits = np.zeros((L, wpr), np.uint64)
    for j in range(L):
        bits[:, j // 64] |= (allowed[:, j].astype(np.uint64) << np.uint64(j % 64))
    mask = fv.Mask.bitmask(torch.from_numpy(bits.view(np.int64)).cuda())
    q, k, v = qkv(13, 1, L, L, 64)
    g = fv.TokenGrid(frames, rows, cols)
    plan = fv.plan_sparse(to_dev(q), to_dev(k), g, g, mask, 3)
    om = oracle.Mask.bitmask(bits)
    refs = oracle_plans(q, k, frames, frames, rows, cols, om, 3)
    _assert_plan_equal(plan, refs)
    out = fv.sparse_attention_exec(to_dev(q), to_dev(k), to_dev(v), plan, mask).float().cpu().numpy()
    ref = oracle_outs(q, k, v, frames, frames, rows, cols, om, refs, oracle.head_scale(64))
    assert rel_l2(out, ref) <= REL_L2_TOL and max_abs(out, ref) <= MAX_ABS_TOL


def test_row_range_and_degenerate_row():
    """Row-range contract (test_sparse.cpp:310-325) and DegenerateRowError (:327-342)."""
    rows = cols = 8
    frames = [0, 1, 2, 3]
    L = 4 * rows * cols
    g = fv.TokenGrid(frames, rows, cols)
    q, k, v = qkv(29, 1, L, L, 64)
    plan = fv.plan_sparse(to_dev(q), to_dev(k), g, g, fv.Mask.all_allowed(), 2)
    full = fv.sparse_attention_exec(to_dev(q), to_dev(k), to_dev(v), plan).float().cpu().numpy()
    tail = fv.sparse_attention_exec(to_dev(q), to_dev(k), to_dev(v), plan, row_begin=128, row_end=L)
    tail = tail.float().cpu().numpy()
    assert np.all(tail[0, :128] == 0)
    np.testing.assert_array_equal(tail[0, 128:], full[0, 128:])
    with pytest.raises(fv.ConfigError):
        fv.sparse_attention_exec(to_dev(q), to_dev(k), to_dev(v), plan, row_begin=10, row_end=5)
    # diagonal-only mask, selections swapped between the two blocks -> no reachable key
    import torch
    wpr = (L + 63) // 64
    bits = np.zeros((L, wpr), np.uint64)
    for i in range(L):
        bits[i, i // 64] |= np.uint64(1) << np.uint64(i % 64)
    mask = fv.Mask.bitmask(torch.from_numpy(bits.view(np.int64)).cuda())
    plan = fv.plan_sparse(to_dev(q), to_dev(k), g, g, mask, 1)
    plan.sel = plan.sel.flip(1).contiguous()
    with pytest.raises(fv.DegenerateRowError):
        fv.sparse_attention_exec(to_dev(q), to_dev(k), to_dev(v), plan, mask)


def test_contract_errors_match_reference_taxonomy():
    g = fv.TokenGrid([0, 1], 16, 16)
    q, k, _ = qkv(1, 1, 512, 512, 64)
    with pytest.raises(fv.ConfigError):
        fv.plan_sparse(to_dev(q), to_dev(k), g, g, fv.Mask.all_allowed(), 0)
    with pytest.raises(fv.ShapeError):
        fv.plan_sparse(to_dev(q[:, :100]), to_dev(k), g, g, fv.Mask.all_allowed(), 2)
    with pytest.raises(fv.ConfigError):
        fv.plan_sparse(to_dev(q), to_dev(k), g, g, fv.Mask.locality(17, 3), 2)
    with pytest.raises(fv.ConfigError):  # frame ids must be strictly increasing (grid.hpp:55)
        fv.plan_sparse(to_dev(q), to_dev(k), fv.TokenGrid([1, 1], 16, 16), g, fv.Mask.all_allowed(), 2)
    bad = q.copy()
    bad[0, :64] = np.inf
    with pytest.raises(fv.ShapeError):
        fv.plan_sparse(to_dev(bad), to_dev(k), g, g, fv.Mask.all_allowed(), 2)


def test_stream_768x1408_step_plan_and_exec():
    """BASELINE config 2: 12 heads, d=128, 48x88 latent, t=32 over {28..32}, k=27."""
    rows, cols, d, heads, topk = 48, 88, 128, 12, 27
    qf, kf = [32], [28, 29, 30, 31, 32]
    N = rows * cols
    q, k, v = qkv(1234, heads, N, 5 * N, d)
    gq, gk = fv.TokenGrid(qf, rows, cols), fv.TokenGrid(kf, rows, cols)
    plan = fv.plan_sparse(to_dev(q), to_dev(k), gq, gk, fv.Mask.all_allowed(), topk)
    check_heads = [0, 7]
    refs = oracle_plans(q[check_heads], k[check_heads], qf, kf, rows, cols, oracle.Mask.all(), topk)
    sel, cnt = plan.sel.cpu().numpy(), plan.count.cpu().numpy()
    for i, h in enumerate(check_heads):
        np.testing.assert_array_equal(sel[h], refs[i].sel)
        np.testing.assert_array_equal(cnt[h], refs[i].count)
    out = fv.sparse_attention_exec(to_dev(q), to_dev(k), to_dev(v), plan).float().cpu().numpy()
    ref = oracle_outs(q[check_heads], k[check_heads], v[check_heads], qf, kf, rows, cols, oracle.Mask.all(), refs,
                      oracle.head_scale(d))
    got = out[check_heads]
    assert rel_l2(got, ref) <= REL_L2_TOL, rel_l2(got, ref)
    assert max_abs(got, ref) <= MAX_ABS_TOL, max_abs(got, ref)


def test_plan_from_fp32_inputs_bit_exact():
    """fvsr_plan_sparse_f32: the reference's own fp32 inputs (not bf16-representable) pooled
    as they are -> indices and coarse-score bits identical to the oracle on the same fp32."""
    import torch
    port = oracle.Port()
    for (qf, kf, rows, cols, d, topk, mask) in [([1], [0, 1], 16, 16, 64, 2, M()),
                                               ([5], [2, 3, 4, 5], 20, 28, 16, 3, M("loc", 7, 9, True)),
                                               ([32], [28, 29, 30, 31, 32], 48, 88, 128, 27, M())]:
        N = rows * cols
        q = port.gaussian(91, len(qf) * N * d).reshape(1, len(qf) * N, d)
        k = port.gaussian(92, len(kf) * N * d).reshape(1, len(kf) * N, d)
        gq, gk = fv.TokenGrid(qf, rows, cols), fv.TokenGrid(kf, rows, cols)
        plan = fv.plan_sparse(torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda(), gq, gk, mask, topk)
        refs = oracle_plans(q, k, qf, kf, rows, cols, to_oracle_mask(mask), topk)
        _assert_plan_equal(plan, refs)
