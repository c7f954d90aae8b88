"""Scored eviction, CPU side: the oracle restatement of
frame_attention_mass (P/src/kv_cache.cpp:170-206) and KVCache::evict (:97-137) pinned to
fixtures produced by the unmodified reference (tests/golden/make_golden_evict.py)."""
import json
import os

import numpy as np
import pytest

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
NPZ = os.path.join(HERE, "golden", "evict_mass.npz")


def golden():
    z = np.load(NPZ)
    meta = json.loads(bytes(z["meta"]).decode())
    return z, meta


def _plan(z, name):
    sel = z[f"{name}.sel"]
    return oracle.Plan(sel, (sel >= 0).sum(1).astype(np.int32), np.zeros(sel.shape[0], np.int32),
                       z[f"{name}.coarse"], z[f"{name}.allowed"])


def _mask(spec):
    return oracle.Mask.all() if spec[0] == "all" else oracle.Mask.locality(spec[1], spec[2], spec[3])


@pytest.mark.parametrize("idx", range(4))
def test_oracle_frame_mass_matches_reference_fixture(idx):
    z, meta = golden()
    c = meta["mass"][idx]
    got = oracle.frame_attention_mass(_plan(z, c["name"]), c["kf"], c["rows"], c["cols"])
    want = z[f"{c['name']}.mass"]
    assert got.dtype == np.float64 and got.shape == (len(c["kf"]),)
    assert np.array_equal(got, want), (got, want)  # bit-exact restatement (libm exp, reference order)
    # the mass is a distribution over q-blocks: it sums to the number of q-blocks with allowed keys
    assert abs(got.sum() - (z[f"{c['name']}.allowed"].any(1)).sum()) < 1e-9


@pytest.mark.parametrize("idx", range(4))
def test_port_plan_reproduces_fixture_scores(idx):
    """The port's plan on the regenerated inputs yields the fixture's coarse scores, so the
    GPU test can feed its own plan into the mass kernel and compare with the fixture."""
    z, meta = golden()
    c = meta["mass"][idx]
    n = c["rows"] * c["cols"]
    q, k, _ = oracle.synthetic_qkv(c["seed"], len(c["qf"]) * n, len(c["kf"]) * n, c["d"])
    p = oracle.Port().plan(q, k, c["qf"], c["kf"], c["rows"], c["cols"], _mask(c["mask"]), c["topk"])
    assert np.array_equal(p.coarse.view(np.uint32), z[f"{c['name']}.coarse"].view(np.uint32))
    assert np.array_equal(p.allowed, z[f"{c['name']}.allowed"])


@pytest.mark.parametrize("idx", range(5))
def test_oracle_evict_matches_reference_fixture(idx):
    z, meta = golden()
    c = meta["evict"][idx]
    kept = oracle.evict(c["strategy"], c["window"], c["ids"], z[f"{c['name']}.scores"], c["heads"])
    want = [[int(i) for i in row if i >= 0] for row in z[f"{c['name']}.kept"]]
    assert kept == want


def test_victims_rule():  # kv_cache.cpp:81-93: newest exempt, lowest first, older on ties
    assert oracle.evict_victims([1, 2, 3, 4], [0.5, 0.1, 0.1, 0.0], 2) == [2, 3]
    assert oracle.evict_victims([1, 2, 3], [0.2, 0.2, 0.0], 5) == [1, 2]


@pytest.mark.skipif(not oracle.ref_available(), reason="reference not built here")
@pytest.mark.parametrize("seed,qf,kf,spec", [(11, [9], [5, 7, 8, 9], ("all",)), (12, [8, 9], [6, 7, 8, 9], ("all",)),
                                             (13, [6], [3, 4, 5, 6], ("loc", 7, 11, False))])
def test_oracle_frame_mass_matches_reference_seeded(seed, qf, kf, spec):
    rows, cols, d = 16, 24, 32
    n = rows * cols
    q, k, v = oracle.synthetic_qkv(seed, len(qf) * n, len(kf) * n, d)
    c = oracle.Ref().case(q, k, v, qf, kf, rows, cols, _mask(spec))
    plan = c.plan(3)
    assert np.array_equal(oracle.frame_attention_mass(plan, kf, rows, cols), c.frame_mass())


# ---- token-mask builders ------------------------------------------------
MASKS = os.path.join(HERE, "golden", "token_masks.npz")
MASK_SIZES = (1, 63, 64, 65, 300, 768)


@pytest.mark.parametrize("L", MASK_SIZES)
def test_oracle_token_masks_match_reference_fixture(L):
    z = np.load(MASKS)
    assert np.array_equal(oracle.segment_mask(z[f"seg{L}.labels"]), z[f"seg{L}.bits"])
    for la in (0, 1):
        assert np.array_equal(oracle.causal_mask(z[f"causal{L}.labels"], la), z[f"causal{L}.la{la}.bits"])


@pytest.mark.parametrize("bad", [[0, 2], [-1, 0], []])
def test_oracle_segment_mask_errors(bad):  # mask.cpp:69-78
    with pytest.raises(oracle.OracleError):
        oracle.segment_mask(bad)


def test_oracle_causal_mask_errors():  # mask.cpp:87-92
    with pytest.raises(oracle.OracleError):
        oracle.causal_mask([1, 0], 0)
    with pytest.raises(oracle.OracleError):
        oracle.causal_mask([0, 1], -1)
