"""Fused RoPE, CPU side: the oracle's apply_rope restatement (P/src/rope.cpp:
30-62) bit-exact against fixtures from the unmodified reference (tests/golden/make_golden_rope.py)."""
import json
import os

import numpy as np
import pytest

import oracle

NPZ = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "rope.npz")


@pytest.mark.parametrize("idx", range(3))
def test_oracle_rope_matches_reference_fixture(idx):
    z = np.load(NPZ)
    c = json.loads(bytes(z["meta"]).decode())[idx]
    L = len(c["fids"]) * c["rows"] * c["cols"]
    x = oracle.bf16_round(oracle.Port().gaussian(c["seed"], L * c["d"]).reshape(L, c["d"]))
    got = oracle.apply_rope(x, c["fids"], c["rows"], c["cols"], c["theta0"], c["split"])
    assert np.array_equal(got.view(np.uint32), z[c["name"]].view(np.uint32))


def test_rope_is_a_rotation():  # pairs keep their norm; position 0 of every axis is the identity
    x = np.random.default_rng(1).standard_normal((64, 64)).astype(np.float32)
    y = oracle.apply_rope(x, [0], 8, 8)
    assert np.array_equal(y[0], x[0])
    n0 = x[:, 0::2] ** 2 + x[:, 1::2] ** 2
    n1 = y[:, 0::2] ** 2 + y[:, 1::2] ** 2
    assert np.allclose(n0, n1, rtol=1e-5)
