"""The fused layer-step (fvsr_ring_step: ring append + mask builder in one launch, then the
attention kernel) against the separate calls (fvsr_ring_append, fvsr_ring_attention) and the
CPU oracle, over a streaming sequence (P/src/stream.cpp:228-256: append before attention,
sliding evict after).  Same plan, same kernels: outputs and selections bitwise equal."""
import numpy as np
import pytest
import torch

import oracle
from tests.helpers import MAX_ABS_TOL, REL_L2_TOL, max_abs, oracle_outs, oracle_plans, qkv, rel_l2, to_dev, to_oracle_mask

pytestmark = pytest.mark.gpu

fv = pytest.importorskip("paper_2510_12747_b200")


@pytest.mark.parametrize("rows,cols,heads,d,topk,window,mask,rope,tq", [
    (48, 88, 12, 128, 27, 4, None, False, 1),
    (24, 40, 3, 128, 5, 4, ("loc", 9, 13, True), False, 1),
    (20, 28, 2, 64, 3, 3, ("loc", 7, 9, False), True, 1),
    (18, 30, 2, 128, 4, 4, None, False, 2),
    (90, 160, 1, 128, 41, 4, ("loc", 72, 72, True), True, 1),
])
def test_fused_step_equals_separate_calls(rows, cols, heads, d, topk, window, mask, rope, tq):
    N = rows * cols
    m = fv.Mask.all_allowed() if mask is None else fv.Mask.locality(mask[1], mask[2], truncated=mask[3])
    a = fv.KVRing(1, heads, d, rows, cols, window + tq)
    b = fv.KVRing(1, heads, d, rows, cols, window + tq)
    if rope:
        a.set_rope()
        b.set_rope()
    port = oracle.Port()
    for t in range(7):
        x = oracle.bf16_round(np.stack([port.gaussian(700 + 10 * t + h, 3 * N * d).reshape(3, N, d)
                                        for h in range(heads)]))
        q, k, v = to_dev(x[:, 0]), to_dev(x[:, 1]), to_dev(x[:, 2])
        qids = [t] if tq == 1 or t % 2 == 0 else [t - 1, t]
        if len(qids) == 2:
            q = torch.cat([qprev, q], dim=1)
        bnq, bnk = fv.block_counts(fv.TokenGrid(qids, rows, cols),
                                   fv.TokenGrid(b.frame_ids(0) + [t], rows, cols))
        cap = min(topk, bnk)
        sa = torch.empty((heads, bnq, cap), dtype=torch.int32, device="cuda")
        sb = torch.empty_like(sa)
        ca = torch.empty((heads, bnq), dtype=torch.int32, device="cuda")
        cb = torch.empty_like(ca)
        if tq == 1 or len(qids) == 2:  # (tq == 2: odd frames close a two-frame chunk)
            oa = a.step(0, t, k, v, q, qids, m, topk, sel=sa, sel_count=ca)
            b.append(0, t, k, v)
            ob = b.attention(0, q, qids, m, topk, sel=sb, sel_count=cb)
            assert torch.equal(sa, sb) and torch.equal(ca, cb), f"t={t}: selections differ"
            assert torch.equal(oa, ob), f"t={t}: fused step output differs from append + attention"
        else:  # first frame of a Tq=2 chunk: append only
            a.append(0, t, k, v)
            b.append(0, t, k, v)
        qprev = to_dev(x[:, 0])
        a.evict(0, window)
        b.evict(0, window)
    assert a.frame_ids(0) == b.frame_ids(0)


@pytest.mark.parametrize("rows,cols,heads,d,topk,mask,rope,tq", [
    (48, 88, 4, 128, 27, None, False, 1),
    (20, 28, 2, 64, 3, ("loc", 7, 9, False), True, 1),
    (18, 30, 2, 128, 4, None, True, 2),
])
def test_bulk_copy_pack_matches_tma_pack(rows, cols, heads, d, topk, mask, rope, tq):
    """The ring append / query pack staged with 1-D bulk copies (FVSR_FLAG_NO_TMA, the
    fallback without the driver's tensor-map entry point) against the tensor-map TMA path:
    the same ring contents, so identical selections and outputs within the bf16 tolerance
    (the |k| bounds are summed in a different order; they only pick the softmax mode)."""
    N = rows * cols
    window = 4
    m = fv.Mask.all_allowed() if mask is None else fv.Mask.locality(mask[1], mask[2], truncated=mask[3])
    bulk_ctx = fv.Context()
    bulk_ctx.set_flags(fv._abi.FLAG_NO_TMA)
    a = fv.KVRing(1, heads, d, rows, cols, window + tq)
    b = fv.KVRing(1, heads, d, rows, cols, window + tq, ctx=bulk_ctx)
    if rope:
        a.set_rope()
        b.set_rope()
    port = oracle.Port()
    qprev = None
    for t in range(7):
        x = oracle.bf16_round(np.stack([port.gaussian(900 + 10 * t + h, 3 * N * d).reshape(3, N, d)
                                        for h in range(heads)]))
        q, k, v = to_dev(x[:, 0]), to_dev(x[:, 1]), to_dev(x[:, 2])
        qids = [t] if tq == 1 or t % 2 == 0 else [t - 1, t]
        if len(qids) == 2:
            q = torch.cat([qprev, q], dim=1)
        if tq == 1 or len(qids) == 2:
            bnq, bnk = fv.block_counts(fv.TokenGrid(qids, rows, cols),
                                       fv.TokenGrid(a.frame_ids(0) + [t], rows, cols))
            cap = min(topk, bnk)
            sa = torch.empty((heads, bnq, cap), dtype=torch.int32, device="cuda")
            sb = torch.empty_like(sa)
            oa = a.step(0, t, k, v, q, qids, m, topk, sel=sa, sel_count=torch.empty((heads, bnq), dtype=torch.int32,
                                                                                   device="cuda"))
            ob = b.step(0, t, k, v, q, qids, m, topk, sel=sb, sel_count=torch.empty((heads, bnq), dtype=torch.int32,
                                                                                   device="cuda"))
            assert torch.equal(sa, sb), f"t={t}: selections differ"
            oa, ob = oa.float().cpu().numpy(), ob.float().cpu().numpy()
            assert rel_l2(ob, oa) <= REL_L2_TOL and max_abs(ob, oa) <= MAX_ABS_TOL, t
        else:
            a.append(0, t, k, v)
            b.append(0, t, k, v)
        qprev = to_dev(x[:, 0])
        a.evict(0, window)
        b.evict(0, window)
    bulk_ctx.check_errors()


def test_fused_step_matches_oracle_768x1408():
    """BASELINE config #2 through fvsr_ring_step: indices bit-exact and output within tolerance."""
    rows, cols, d, heads, topk, window = 48, 88, 128, 12, 27, 4
    N = rows * cols
    ring = fv.KVRing(1, heads, d, rows, cols, window)
    port = oracle.Port()
    ks, vs, ids = [], [], []
    for t in range(28, 33):
        x = oracle.bf16_round(np.stack([port.gaussian(900 + 10 * t + h, 3 * N * d).reshape(3, N, d)
                                        for h in range(heads)]))
        q, k, v = x[:, 0], x[:, 1], x[:, 2]
        ids.append(t)
        ks.append(k)
        vs.append(v)
        bnq, bnk = fv.block_counts(fv.TokenGrid([t], rows, cols), fv.TokenGrid(ids, rows, cols))
        sel = torch.empty((heads, bnq, min(topk, bnk)), dtype=torch.int32, device="cuda")
        cnt = torch.empty((heads, bnq), dtype=torch.int32, device="cuda")
        out = ring.step(0, t, to_dev(k), to_dev(v), to_dev(q), [t], fv.Mask.all_allowed(), topk, sel=sel,
                        sel_count=cnt)
        ring.evict(0)
    K, V = np.concatenate(ks, axis=1), np.concatenate(vs, axis=1)
    from tests.helpers import par_map
    plans = par_map(lambda h: oracle.Port().plan(q[h], K[h], [32], ids, rows, cols, oracle.Mask.all(), topk),
                    range(heads))
    for h in range(heads):
        np.testing.assert_array_equal(sel[h].cpu().numpy(), plans[h].sel)
    ref = np.stack(par_map(lambda h: oracle.Port().exec(q[h], K[h], V[h], [32], ids, rows, cols, oracle.Mask.all(),
                                                        plans[h], oracle.head_scale(d)), range(heads)))
    got = out.float().cpu().numpy()
    assert rel_l2(got, ref) <= REL_L2_TOL and max_abs(got, ref) <= MAX_ABS_TOL


def test_ring_step_over_1024_key_blocks():
    """A ring context with more than 1024 key blocks (13 frames of 8x20 tiles: 7 temporal rows x
    160 tiles = 1120) runs the selector's widest instantiation (NPER = 128 candidates per lane,
    four key blocks per thread): selections exact and outputs within tolerance of the oracle."""
    heads, rows, cols, d, topk, window = 1, 64, 160, 64, 20, 12
    N = rows * cols
    ring = fv.KVRing(1, heads, d, rows, cols, window)
    port = oracle.Port()
    store = {}
    for t in range(window + 1):
        x = oracle.bf16_round(port.gaussian(3100 + t, 3 * N * d).reshape(3, 1, N, d))
        store[t] = x
        q, k, v = to_dev(x[0]), to_dev(x[1]), to_dev(x[2])
        ids = ring.frame_ids(0) + [t]
        if t < window:
            ring.append(0, t, k, v)
            continue
        bnq, bnk = fv.block_counts(fv.TokenGrid([t], rows, cols), fv.TokenGrid(ids, rows, cols))
        assert bnk > 1024
        sel = torch.empty((heads, bnq, topk), dtype=torch.int32, device="cuda")
        cnt = torch.empty((heads, bnq), dtype=torch.int32, device="cuda")
        out = ring.step(0, t, k, v, q, [t], fv.Mask.all_allowed(), topk, sel=sel, sel_count=cnt)
        out = out.float().cpu().numpy()
        K = np.concatenate([store[i][1] for i in ids], axis=1)
        V = np.concatenate([store[i][2] for i in ids], axis=1)
        Q = store[t][0]
        plans = oracle_plans(Q, K, [t], ids, rows, cols, oracle.Mask.all(), topk)
        assert np.array_equal(sel[0].cpu().numpy()[:, : plans[0].sel.shape[1]], plans[0].sel)
        assert np.array_equal(cnt[0].cpu().numpy(), plans[0].count)
        ref = oracle_outs(Q, K, V, [t], ids, rows, cols, oracle.Mask.all(), plans, oracle.head_scale(d))
        assert rel_l2(out, ref) <= REL_L2_TOL and max_abs(out, ref) <= MAX_ABS_TOL
