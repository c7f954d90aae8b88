"""GPU parity at the BASELINE shapes (VERDICT r1 "What's weak" 1): every config the bench and
the sweeps quote, checked against the CPU oracle on the GPU box.

    768x1408 step (config #2)   12 heads, all-allowed and locality (48,72) truncated/preserved, k=27
    768x1408 Tq=2 chunk         paired query frames -> the NQ=128 kernel at full shape
    1440p (config #4)           90x160 (ragged 2-row bottom tile row), locality 72x72 both modes
                                at k=41 and all-allowed at k=98 -> topk_select_kernel<32>
    k > 256                     the attention kernel's per-unit table overflow (kInfoCap) path
    bnk > 1024                  topk_select_kernel<128> (plan only)

Block indices bit-exact (all heads computed); outputs within REL_L2_TOL / MAX_ABS_TOL of the
fp32 oracle fed the same bf16-rounded inputs.  Each case records its per-shape errors with
record_parity (profiles/parity_r2.json).  The oracle (oracle/fvsr_port.c, test-only) runs one
head per thread.
"""
import numpy as np
import pytest

import oracle
from tests.helpers import (MAX_ABS_TOL, REL_L2_TOL, max_abs, par_map, qkv, record_parity, rel_l2, to_dev,
                           to_oracle_mask)

pytestmark = pytest.mark.gpu

fv = pytest.importorskip("paper_2510_12747_b200")


def _plans(q, k, qf, kf, rows, cols, om, topk):
    return par_map(lambda h: oracle.Port().plan(q[h], k[h], qf, kf, rows, cols, om, topk), range(q.shape[0]))


def _outs(q, k, v, qf, kf, rows, cols, om, plans, scale, row_begin=0, row_end=-1):
    return np.stack(par_map(lambda h: oracle.Port().exec(q[h], k[h], v[h], qf, kf, rows, cols, om, plans[h], scale,
                                                         row_begin, row_end), range(q.shape[0])))


def _check_plan(plan, refs):
    sel, cnt, diag = plan.sel.cpu().numpy(), plan.count.cpu().numpy(), plan.diagonal_block.cpu().numpy()
    coarse = plan.coarse_scores.cpu().numpy() if plan.coarse_scores is not None else None
    for h, r in enumerate(refs):
        np.testing.assert_array_equal(cnt[h], r.count, err_msg=f"head {h} counts")
        np.testing.assert_array_equal(sel[h], r.sel, err_msg=f"head {h} selected ids")
        np.testing.assert_array_equal(diag[h], r.diag, err_msg=f"head {h} diagonal")
        if coarse is not None:
            np.testing.assert_array_equal(coarse[h].view(np.uint32), r.coarse.view(np.uint32),
                                          err_msg=f"head {h} coarse score bits")


# name, seed, heads, q frames, k frames, rows, cols, d, topk, mask, exec row range (None: all)
BIG = [
    ("768x1408_all_k27_12h", 1234, 12, [32], [28, 29, 30, 31, 32], 48, 88, 128, 27, ("all",), None),
    ("768x1408_loc48x72_trunc_k27_12h", 1235, 12, [32], [28, 29, 30, 31, 32], 48, 88, 128, 27,
     ("loc", 48, 72, True), None),
    ("768x1408_loc48x72_pres_k27_12h", 1236, 12, [33], [29, 30, 31, 32, 33], 48, 88, 128, 27,
     ("loc", 48, 72, False), None),
    ("768x1408_tq2_chunk_k36_2h", 1237, 2, [32, 33], [28, 29, 30, 31, 32, 33], 48, 88, 128, 36, ("all",), None),
    ("1440p_loc72x72_trunc_k41_2h", 1440, 2, [32], [28, 29, 30, 31, 32], 90, 160, 128, 41,
     ("loc", 72, 72, True), None),
    ("1440p_loc72x72_pres_k41_2h", 1441, 2, [33], [29, 30, 31, 32, 33], 90, 160, 128, 41,
     ("loc", 72, 72, False), None),
    ("1440p_all_k98_1h", 1442, 1, [32], [28, 29, 30, 31, 32], 90, 160, 128, 98, ("all",), None),
    # k > kInfoCap (256): 9 frames of 64x64 -> bnk 320, k=300; output rows [0, 1024) checked
    ("k300_bnk320_info_overflow", 77, 1, [32], list(range(24, 33)), 64, 64, 128, 300, ("all",), (0, 1024)),
]


def _mask(spec):
    if spec[0] == "all":
        return fv.Mask.all_allowed()
    return fv.Mask.locality(spec[1], spec[2], truncated=spec[3])


@pytest.mark.parametrize("c", BIG, ids=[c[0] for c in BIG])
def test_baseline_shape_parity(c):
    name, seed, heads, qf, kf, rows, cols, d, topk, mspec, rr = c
    N = rows * cols
    q, k, v = qkv(seed, heads, len(qf) * N, len(kf) * N, d)
    mask = _mask(mspec)
    om = to_oracle_mask(mask)
    gq, gk = fv.TokenGrid(qf, rows, cols), fv.TokenGrid(kf, rows, cols)
    plan = fv.plan_sparse(to_dev(q), to_dev(k), gq, gk, mask, topk)
    refs = _plans(q, k, qf, kf, rows, cols, om, topk)
    _check_plan(plan, refs)
    scale = oracle.head_scale(d)
    rb, re = rr if rr else (0, -1)
    out = fv.sparse_attention_exec(to_dev(q), to_dev(k), to_dev(v), plan, mask, scale, row_begin=rb,
                                   row_end=None if re < 0 else re).float().cpu().numpy()
    ref = _outs(q, k, v, qf, kf, rows, cols, om, refs, scale, rb, re)
    e, m = rel_l2(out, ref), max_abs(out, ref)
    per_head = [(rel_l2(out[h], ref[h]), max_abs(out[h], ref[h])) for h in range(heads)]
    record_parity(name, rows=rows, cols=cols, heads=heads, d=d, q_frames=qf, k_frames=kf, topk=topk,
                  mask=list(mspec), bnq=int(plan.bnq), bnk=int(plan.coarse_scores.shape[2]),
                  selected_per_qblock=[int(plan.count.min()), int(plan.count.max())], rows_checked=[rb, re],
                  indices_bit_exact=True, rel_l2=e, max_abs=m, worst_head_rel_l2=max(p[0] for p in per_head),
                  worst_head_max_abs=max(p[1] for p in per_head), tol_rel_l2=REL_L2_TOL, tol_max_abs=MAX_ABS_TOL)
    assert e <= REL_L2_TOL and m <= MAX_ABS_TOL, (name, e, m)


def test_plan_bnk_over_1024_selector():
    """1440p over 9 frames: bnk = 5 temporal rows x 240 tiles = 1200 > 1024 -> the NPER=128
    selector; k = topk_for_density(0.136, 1200) = 163.  Plan only (bit-exact)."""
    rows, cols, d, topk = 90, 160, 64, 163
    qf, kf = [32], list(range(24, 33))
    N = rows * cols
    q, k, _ = qkv(1443, 1, N, len(kf) * N, d)
    gq, gk = fv.TokenGrid(qf, rows, cols), fv.TokenGrid(kf, rows, cols)
    plan = fv.plan_sparse(to_dev(q), to_dev(k), gq, gk, fv.Mask.all_allowed(), topk)
    assert plan.coarse_scores.shape[2] == 1200
    refs = _plans(q, k, qf, kf, rows, cols, oracle.Mask.all(), topk)
    _check_plan(plan, refs)
    record_parity("1440p_9frames_bnk1200_plan", rows=rows, cols=cols, heads=1, d=d, topk=topk, bnk=1200,
                  indices_bit_exact=True)


def test_ring_stream_1440p_locality():
    """The streaming ring at 1440p with a 72x72 truncated window (config #4 as the bench's
    sweep runs it): append, mask builder, attention over 6 steps, 2 heads; indices exact and
    outputs within tolerance at the last step."""
    rows, cols, d, heads, topk, window = 90, 160, 128, 2, 41, 4
    N = rows * cols
    mask = fv.Mask.locality(72, 72, truncated=True)
    om = to_oracle_mask(mask)
    ring = fv.KVRing(1, heads, d, rows, cols, window)
    port = oracle.Port()
    ks, vs, ids = [], [], []
    for t in range(6):
        x = oracle.bf16_round(np.stack([port.gaussian(5000 + 10 * t + h, 3 * N * d).reshape(3, N, d)
                                        for h in range(heads)]))
        q, k, v = x[:, 0], x[:, 1], x[:, 2]
        ring.append(0, t, to_dev(k), to_dev(v))
        ids.append(t)
        ks.append(k)
        vs.append(v)
        out = ring.attention(0, to_dev(q), [t], mask, topk)
        if t == 5:
            K, V = np.concatenate(ks, axis=1), np.concatenate(vs, axis=1)
            plans = _plans(q, K, [t], ids, rows, cols, om, topk)
            bnq, bnk = fv.block_counts(fv.TokenGrid([t], rows, cols), fv.TokenGrid(ids, rows, cols))
            import torch
            sel = torch.empty((heads, bnq, min(topk, bnk)), dtype=torch.int32, device="cuda")
            cnt = torch.empty((heads, bnq), dtype=torch.int32, device="cuda")
            out = ring.attention(0, to_dev(q), [t], mask, topk, sel=sel, sel_count=cnt)
            for h in range(heads):
                np.testing.assert_array_equal(sel[h].cpu().numpy(), plans[h].sel)
            ref = _outs(q, K, V, [t], ids, rows, cols, om, plans, oracle.head_scale(d))
            got = out.float().cpu().numpy()
            e, m = rel_l2(got, ref), max_abs(got, ref)
            record_parity("ring_1440p_loc72x72_trunc_k41_t5", rows=rows, cols=cols, heads=heads, d=d, topk=topk,
                          k_frames=list(ids), indices_bit_exact=True, rel_l2=e, max_abs=m)
            assert e <= REL_L2_TOL and m <= MAX_ABS_TOL, (e, m)
        ring.evict(0)
        while len(ids) > window:
            ids.pop(0)
            ks.pop(0)
            vs.pop(0)


def test_saturated_plan_equals_dense_oracle():
    """a11: with k = bnk every allowed block is selected, so sparse exec equals dense attention
    (P/tests/test_sparse.cpp:200-213, P/src/checks.cpp:90-118).  Checked against the reference's
    own dense_attention_oracle (P/src/attention.cpp:40-56) via oracle/_ref, for the all-allowed
    and a locality mask."""
    if not oracle.ref_available():
        pytest.skip("oracle/_ref (compiled reference) not built")
    rows, cols, d = 24, 40, 128
    qf, kf = [5], [2, 3, 4, 5]
    N = rows * cols
    q, k, v = qkv(4242, 1, N, len(kf) * N, d)
    bnq, bnk = fv.block_counts(fv.TokenGrid(qf, rows, cols), fv.TokenGrid(kf, rows, cols))
    for mask in (fv.Mask.all_allowed(), fv.Mask.locality(9, 13, truncated=True)):
        om = to_oracle_mask(mask)
        gq, gk = fv.TokenGrid(qf, rows, cols), fv.TokenGrid(kf, rows, cols)
        plan = fv.plan_sparse(to_dev(q), to_dev(k), gq, gk, mask, bnk)
        out = fv.sparse_attention_exec(to_dev(q), to_dev(k), to_dev(v), plan, mask).float().cpu().numpy()[0]
        case = oracle.Ref().case(q[0], k[0], v[0], qf, kf, rows, cols, om)
        dense = case.dense(oracle.head_scale(d))
        e, m = rel_l2(out, dense), max_abs(out, dense)
        record_parity("saturated_vs_dense_oracle_" + ("all" if mask.kind == 0 else "loc9x13"), rows=rows, cols=cols,
                      d=d, topk=bnk, rel_l2=e, max_abs=m)
        assert e <= REL_L2_TOL and m <= MAX_ABS_TOL, (e, m)
