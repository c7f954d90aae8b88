"""GPU fused RoPE: fvsr_ring_set_rope makes the ring's pack/pool pass apply
apply_rope (P/src/rope.cpp:30-62) to K on append and to Q in the mask builder, at absolute
(frame, row, col) positions, as make_frame_kv / step do (P/src/stream.cpp:134-152, 240).

Parity: the ring is fed un-rotated bf16 projections; the oracle rotates them with its
reference-pinned apply_rope and rounds to bf16 (what the device stores).  Block indices
bit-exact every step, outputs within the bf16 tolerance."""
import numpy as np
import pytest
import torch

import oracle
from tests.helpers import MAX_ABS_TOL, REL_L2_TOL, max_abs, oracle_outs, oracle_plans, rel_l2, to_dev

pytestmark = pytest.mark.gpu
fv = pytest.importorskip("paper_2510_12747_b200")


@pytest.mark.parametrize("d,rows,cols,split,theta0,start", [(128, 16, 40, None, 10000.0, 0),
                                                            (64, 20, 28, [16, 32, 16], 500.0, 37),
                                                            (128, 12, 20, None, 10000.0, 1000)])
def test_ring_rope_matches_oracle(d, rows, cols, split, theta0, start):
    heads, topk, window = 2, 4, 3
    n = rows * cols
    ring = fv.KVRing(1, heads, d, rows, cols, window)
    ring.set_rope(theta0, split)
    port = oracle.Port()
    kr, vs, ids = {}, {}, []
    tiles = ((rows + 7) // 8) * ((cols + 7) // 8)
    for t in range(start, start + 6):
        x = oracle.bf16_round(np.stack([port.gaussian(1300 + 10 * t + h, 3 * n * d).reshape(3, n, d)
                                        for h in range(heads)]))
        q, k, v = x[:, 0], x[:, 1], x[:, 2]
        ring.append(0, t, to_dev(k), to_dev(v))
        ids.append(t)
        qr = np.stack([oracle.bf16_round(oracle.apply_rope(q[h], [t], rows, cols, theta0, split)) for h in range(heads)])
        kr[t] = np.stack([oracle.bf16_round(oracle.apply_rope(k[h], [t], rows, cols, theta0, split))
                          for h in range(heads)])
        vs[t] = v
        sel = torch.empty((heads, tiles, topk), dtype=torch.int32, device="cuda")
        cnt = torch.empty((heads, tiles), dtype=torch.int32, device="cuda")
        out = ring.attention(0, to_dev(q), [t], fv.Mask.all_allowed(), topk, sel=sel, sel_count=cnt)
        out = out.float().cpu().numpy()
        K = np.concatenate([kr[i] for i in ids], axis=1)
        V = np.concatenate([vs[i] for i in ids], axis=1)
        plans = oracle_plans(qr, K, [t], ids, rows, cols, oracle.Mask.all(), topk)
        ref = oracle_outs(qr, K, V, [t], ids, rows, cols, oracle.Mask.all(), plans, oracle.head_scale(d))
        for h in range(heads):
            assert np.array_equal(sel[h].cpu().numpy()[:, : plans[h].sel.shape[1]], plans[h].sel), (t, h)
        assert rel_l2(out, ref) <= REL_L2_TOL and max_abs(out, ref) <= MAX_ABS_TOL, (rel_l2(out, ref),
                                                                                     max_abs(out, ref))
        ring.evict(0)
        while len(ids) > window:
            ids.pop(0)


def test_ring_rope_two_query_frames():
    """Chunked streaming (Tq=2): both query frames rotated at their own frame ids."""
    heads, rows, cols, d, topk, window = 2, 16, 24, 128, 4, 3
    n = rows * cols
    ring = fv.KVRing(1, heads, d, rows, cols, window + 1)
    ring.set_rope()
    port = oracle.Port()
    ks, vs, qs = [], [], []
    fids = [4, 5]
    for t in fids:
        x = oracle.bf16_round(np.stack([port.gaussian(1500 + 10 * t + h, 3 * n * d).reshape(3, n, d)
                                        for h in range(heads)]))
        ring.append(0, t, to_dev(x[:, 1]), to_dev(x[:, 2]))
        qs.append(x[:, 0]); ks.append(x[:, 1]); vs.append(x[:, 2])
    q = np.concatenate(qs, axis=1)
    out = ring.attention(0, to_dev(q), fids, fv.Mask.all_allowed(), topk).float().cpu().numpy()
    rot = lambda a: np.stack([oracle.bf16_round(oracle.apply_rope(a[h], fids, rows, cols)) for h in range(heads)])
    qr, K, V = rot(q), rot(np.concatenate(ks, axis=1)), np.concatenate(vs, axis=1)
    plans = oracle_plans(qr, K, fids, fids, rows, cols, oracle.Mask.all(), topk)
    ref = oracle_outs(qr, K, V, fids, fids, rows, cols, oracle.Mask.all(), plans, oracle.head_scale(d))
    assert rel_l2(out, ref) <= REL_L2_TOL and max_abs(out, ref) <= MAX_ABS_TOL


def test_set_rope_errors():  # RopeConfig::validate (P/src/rope.cpp:19-28)
    ring = fv.KVRing(1, 1, 64, 8, 8, 2)
    with pytest.raises(fv.ConfigError):
        ring.set_rope(10000.0, [16, 16, 16])
    with pytest.raises(fv.ConfigError):
        ring.set_rope(10000.0, [31, 17, 16])
    with pytest.raises(fv.ConfigError):
        ring.set_rope(1.0)
