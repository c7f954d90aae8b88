"""GPU parity of scored eviction: fvsr_frame_attention_mass /
fvsr_ring_frame_mass (frame_attention_mass, P/src/kv_cache.cpp:170-206) against the
reference fixtures and the oracle, and fvsr_ring_evict (KVCache::evict, :97-137) driving a
streaming ring whose retained frames become non-contiguous.

Tolerance: masses within 1e-12 relative (device exp and reduction order differ from libm /
the reference's sequential sums in the last ulps); retained frame sets and block indices
exact."""
import json
import os

import numpy as np
import torch
import pytest

import oracle
from tests.helpers import MAX_ABS_TOL, REL_L2_TOL, max_abs, oracle_outs, oracle_plans, rel_l2, to_dev

pytestmark = pytest.mark.gpu
fv = pytest.importorskip("paper_2510_12747_b200")

MASS_RTOL = 1e-12
NPZ = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "evict_mass.npz")


def _masks(spec):
    if spec[0] == "all":
        return fv.Mask.all_allowed(), oracle.Mask.all()
    return fv.Mask.locality(spec[1], spec[2], spec[3]), oracle.Mask.locality(spec[1], spec[2], spec[3])


def _close(got, want):
    return np.all(np.abs(got - want) <= MASS_RTOL * np.maximum(np.abs(want), 1.0))


@pytest.mark.parametrize("idx", range(4))
def test_frame_mass_matches_reference_fixture(idx):
    z = np.load(NPZ)
    c = json.loads(bytes(z["meta"]).decode())["mass"][idx]
    n = c["rows"] * c["cols"]
    q, k, _ = oracle.synthetic_qkv(c["seed"], len(c["qf"]) * n, len(c["kf"]) * n, c["d"])
    fmask, _ = _masks(c["mask"])
    gq, gk = fv.TokenGrid(c["qf"], c["rows"], c["cols"]), fv.TokenGrid(c["kf"], c["rows"], c["cols"])
    plan = fv.plan_sparse(to_dev(q[None]), to_dev(k[None]), gq, gk, fmask, c["topk"])
    assert np.array_equal(plan.coarse_scores[0].cpu().numpy().view(np.uint32), z[f"{c['name']}.coarse"].view(np.uint32))
    mass = fv.frame_attention_mass(plan, gk, fmask).cpu().numpy()[0]
    want = z[f"{c['name']}.mass"]
    assert _close(mass, want), (mass, want)


def test_frame_mass_multi_head_matches_oracle():
    heads, rows, cols, d, qf, kf = 3, 24, 32, 128, [9], [5, 7, 8, 9]
    n = rows * cols
    port = oracle.Port()
    x = oracle.bf16_round(np.stack([port.gaussian(700 + h, (1 + 2 * len(kf)) * n * d) for h in range(heads)]))
    q = x[:, : n * d].reshape(heads, n, d)
    k = x[:, n * d: n * d + len(kf) * n * d].reshape(heads, len(kf) * n, d)
    gq, gk = fv.TokenGrid(qf, rows, cols), fv.TokenGrid(kf, rows, cols)
    plan = fv.plan_sparse(to_dev(q), to_dev(k), gq, gk, fv.Mask.all_allowed(), 6)
    mass = fv.frame_attention_mass(plan).cpu().numpy()
    for h in range(heads):
        p = port.plan(q[h], k[h], qf, kf, rows, cols, oracle.Mask.all(), 6)
        assert _close(mass[h], oracle.frame_attention_mass(p, kf, rows, cols))


@pytest.mark.parametrize("strategy,mask", [(1, None), (1, ("loc", 9, 13, True)), (2, None)])
def test_streaming_ring_scored_eviction(strategy, mask):
    """step()-style loop (P/src/stream.cpp:237-266): append, attention, frame scores from the
    plan, evict with the scored strategy.  The ring's retained set, the selection and the
    outputs track the oracle every step, including after non-contiguous evictions."""
    heads, rows, cols, d, topk, window = 2, 16, 40, 128, 4, 3
    n = rows * cols
    fmask, omask = _masks(mask or ("all",))
    ring = fv.KVRing(1, heads, d, rows, cols, window)
    port = oracle.Port()
    store = {}
    ids = []
    saw_gap = False
    for t in range(10):
        x = oracle.bf16_round(np.stack([port.gaussian(800 + 10 * t + h, 3 * n * d).reshape(3, n, d)
                                        for h in range(heads)]))
        q, k, v = x[:, 0], x[:, 1], x[:, 2]
        if strategy == 2:  # identical heads -> identical head-wise decisions (the ring keeps shared sets)
            q, k, v = np.repeat(q[:1], heads, 0), np.repeat(k[:1], heads, 0), np.repeat(v[:1], heads, 0)
        ring.append(0, t, to_dev(k), to_dev(v))
        store[t] = (k, v)
        ids.append(t)
        assert ring.frame_ids(0) == ids
        saw_gap |= any(b - a > 1 for a, b in zip(ids, ids[1:]))
        sel = torch.empty((heads, (rows // 8) * (cols // 8), topk), dtype=torch.int32,
                                        device="cuda")
        cnt = torch.empty((heads, sel.shape[1]), dtype=torch.int32, device="cuda")
        out = ring.attention(0, to_dev(q), [t], fmask, topk, sel=sel, sel_count=cnt).float().cpu().numpy()
        mass = ring.frame_mass(0, [t], fmask).cpu().numpy()
        K = np.concatenate([store[i][0] for i in ids], axis=1)
        V = np.concatenate([store[i][1] for i in ids], axis=1)
        plans = oracle_plans(q, K, [t], ids, rows, cols, omask, topk)
        ref = oracle_outs(q, K, V, [t], ids, rows, cols, omask, plans, oracle.head_scale(d))
        assert rel_l2(out, ref) <= REL_L2_TOL and max_abs(out, ref) <= MAX_ABS_TOL
        want_mass = np.stack([oracle.frame_attention_mass(p, ids, rows, cols) for p in plans])
        for h in range(heads):
            assert np.array_equal(sel[h].cpu().numpy()[:, : plans[h].sel.shape[1]], plans[h].sel)
            assert _close(mass[h], want_mass[h]), (t, h, mass[h], want_mass[h])
        ring.evict_scored(0, strategy, mass)
        kept = oracle.evict(strategy, window, ids, want_mass, heads)
        ids = kept[0]
        assert ring.frame_ids(0) == ids, (t, ring.frame_ids(0), ids)
    assert saw_gap or strategy == 2  # uniform eviction must have produced a non-contiguous context


def test_ring_evict_errors():
    ring = fv.KVRing(1, 2, 64, 8, 16, 2)
    for t in range(3):
        ring.append(0, t, to_dev(np.zeros((2, 128, 64), np.float32)), to_dev(np.zeros((2, 128, 64), np.float32)))
    with pytest.raises(fv.ConfigError):  # scores required while over budget (kv_cache.cpp:112-113)
        ring.evict_scored(0, fv.EVICT_UNIFORM, None)
    with pytest.raises(fv.ShapeError):
        ring.evict_scored(0, fv.EVICT_UNIFORM, np.zeros((2, 2)))
    with pytest.raises(fv.ConfigError):  # no scores of this layer-step on the context
        fv.KVRing(1, 2, 64, 8, 16, 2).frame_mass(0, [0])
    ring.evict_scored(0, fv.EVICT_UNIFORM, np.array([[0.0, 1.0, 2.0], [0.5, 0.0, 2.0]]))
    assert ring.frame_ids(0) == [1, 2]
    # head-wise victims that differ across heads: the sets diverge (kv_cache.cpp:130-136)
    ring2 = fv.KVRing(1, 2, 64, 8, 16, 2)
    for t in range(3):
        ring2.append(0, t, to_dev(np.zeros((2, 128, 64), np.float32)), to_dev(np.zeros((2, 128, 64), np.float32)))
    ring2.evict_scored(0, fv.EVICT_HEAD_WISE, np.array([[0.0, 1.0, 2.0], [1.0, 0.0, 2.0]]))
    assert ring2.frame_ids_head(0, 0) == [1, 2] and ring2.frame_ids_head(0, 1) == [0, 2]


@pytest.mark.parametrize("mask", [None, ("loc", 9, 13, True)])
def test_headwise_eviction_diverging_heads(mask):
    """KVCache::evict(head_wise) with heads that pick DIFFERENT victims (P/src/kv_cache.cpp:
    130-136): each head keeps its own frame table, later steps run one launch per run of heads
    with identical sets, and every head's selection, output and frame masses track the oracle
    run on that head's own context; the retained sets diverge at least once."""
    heads, rows, cols, d, topk, window = 4, 16, 40, 128, 4, 3
    n = rows * cols
    fmask, omask = _masks(mask or ("all",))
    ring = fv.KVRing(1, heads, d, rows, cols, window)
    port = oracle.Port()
    store = {}
    ids = [[] for _ in range(heads)]
    diverged = False
    for t in range(12):
        x = oracle.bf16_round(np.stack([port.gaussian(1300 + 10 * t + h, 3 * n * d).reshape(3, n, d)
                                        for h in range(heads)]))
        q, k, v = x[:, 0], x[:, 1], x[:, 2]
        store[t] = (k, v)
        for h in range(heads):
            ids[h].append(t)
        bnq = (rows // 8) * (cols // 8)
        sel = torch.empty((heads, bnq, topk), dtype=torch.int32, device="cuda")
        cnt = torch.empty((heads, bnq), dtype=torch.int32, device="cuda")
        out = ring.step(0, t, to_dev(k), to_dev(v), to_dev(q), [t], fmask, topk, sel=sel, sel_count=cnt)
        out = out.float().cpu().numpy()
        mass = ring.frame_mass(0, [t], fmask).cpu().numpy()
        for h in range(heads):
            assert ring.frame_ids_head(0, h) == ids[h], (t, h)
            K = np.concatenate([store[i][0][h] for i in ids[h]], axis=0)
            V = np.concatenate([store[i][1][h] for i in ids[h]], axis=0)
            p = port.plan(q[h], K, [t], ids[h], rows, cols, omask, topk)
            assert np.array_equal(sel[h].cpu().numpy()[:, : p.sel.shape[1]], p.sel), (t, h)
            ref = port.exec(q[h], K, V, [t], ids[h], rows, cols, omask, p, oracle.head_scale(d))
            assert rel_l2(out[h], ref) <= REL_L2_TOL and max_abs(out[h], ref) <= MAX_ABS_TOL, (t, h)
            assert _close(mass[h], oracle.frame_attention_mass(p, ids[h], rows, cols)), (t, h)
        ring.evict_scored(0, fv.EVICT_HEAD_WISE, mass)
        for h in range(heads):
            if len(ids[h]) > window:
                gone = set(oracle.evict_victims(ids[h], list(mass[h]), len(ids[h]) - window))
                ids[h] = [i for i in ids[h] if i not in gone]
            assert ring.frame_ids_head(0, h) == ids[h], (t, h)
        diverged |= any(ids[h] != ids[0] for h in range(heads))
    assert diverged
    if any(ids[h] != ids[0] for h in range(heads)):  # uniform needs head-identical sets (kv_cache.cpp:119-122)
        ring.append(0, 12, to_dev(store[11][0]), to_dev(store[11][1]))
        with pytest.raises(fv.InvariantError):
            ring.evict_scored(0, fv.EVICT_UNIFORM, np.ones((heads, ring.retained(0))))
