"""The streaming toy-DiT step on the GPU (P/src/stream.cpp:198-281):
RMSNorm kernel, K/V projection read in place by the ring append (fvsr_ring_step_layout: the
per-head split and RoPE fused into the append), Q RoPE + mask builder + attention writing
[tokens][D] for the output projection, FFN, sliding eviction -- over several streamed frames.

Checked per (frame, layer) from the step's recorded intermediates:
  * rms_norm against the reference formula (double accumulation) -> bf16 rounding;
  * the attention output against the CPU oracle given the step's own bf16 projections (RoPE
    by the reference-pinned oracle.apply_rope, plan + exec by the oracle over the ring's
    retained frames) within the bf16 tolerance;
  * the residual updates (x += att Wo; x += silu(rms(x) W_in) W_out) recomputed in fp32.
"""
import numpy as np
import pytest
import torch

import oracle
from tests.helpers import MAX_ABS_TOL, REL_L2_TOL, max_abs, rel_l2

pytestmark = pytest.mark.gpu

fv = pytest.importorskip("paper_2510_12747_b200")
from paper_2510_12747_b200.toy_dit import StreamDiTConfig, StreamingDiT  # noqa: E402


def _rms_ref(x, g):
    x = x.astype(np.float64)
    inv = 1.0 / np.sqrt((x * x).mean(axis=1, keepdims=True) + 1e-6)
    return (x.astype(np.float32) * inv.astype(np.float32) * g.astype(np.float32)).astype(np.float32)


@pytest.mark.parametrize("mask", [None, ("loc", 9, 11, True)])
def test_streaming_dit_layer_loop(mask):
    m = None if mask is None else fv.Mask.locality(mask[1], mask[2], truncated=mask[3])
    cfg = StreamDiTConfig(n_layers=2, n_heads=2, d_head=64, ffw_dim=128, latent_rows=16, latent_cols=24,
                          window_frames=3, topk=3, mask=m)
    dit = StreamingDiT(cfg)
    N, D, d, H = cfg.tokens_per_frame, cfg.model_dim, cfg.d_head, cfg.n_heads
    om = oracle.Mask.all() if m is None else oracle.Mask.locality(mask[1], mask[2], truncated=mask[3])
    gen = torch.Generator(device="cuda").manual_seed(5)
    hist = {l: [] for l in range(cfg.n_layers)}  # per layer: (frame id, K_rot [H, N, d], V [H, N, d])
    port = oracle.Port()
    for t in range(6):
        x0 = torch.randn((N, D), generator=gen, device="cuda")
        dit.trace = []
        x_out = dit.step(x0)
        for rec in dit.trace:
            l, w = rec["layer"], dit.layers[rec["layer"]]
            x = rec["x"].cpu().numpy()
            # rms_norm kernel vs the reference formula (the Q operand)
            xn = dit.rms_norm(rec["x"], w.norm1_g).float().cpu().numpy()
            ref_xn = oracle.bf16_round(_rms_ref(x, w.norm1_g.cpu().numpy()))
            assert max_abs(xn, ref_xn) <= 2 * 2.0 ** -8 * np.abs(ref_xn).max(), l
            # attention from the step's own projections
            kv = rec["kv"].float().cpu().numpy()
            q = rec["q"].float().cpu().numpy()
            k_rot = np.stack([oracle.bf16_round(oracle.apply_rope(kv[:, h * d:(h + 1) * d], [t], cfg.latent_rows,
                                                                  cfg.latent_cols)) for h in range(H)])
            v = np.stack([kv[:, D + h * d:D + (h + 1) * d] for h in range(H)])
            q_rot = np.stack([oracle.bf16_round(oracle.apply_rope(q[:, h * d:(h + 1) * d], [t], cfg.latent_rows,
                                                                  cfg.latent_cols)) for h in range(H)])
            hist[l].append((t, k_rot, v))
            hist[l] = hist[l][-(cfg.window_frames + 1):]
            ids = [f for f, _, _ in hist[l]]
            K = np.concatenate([k for _, k, _ in hist[l]], axis=1)
            V = np.concatenate([vv for _, _, vv in hist[l]], axis=1)
            att = rec["att"].float().cpu().numpy()
            for h in range(H):
                plan = port.plan(q_rot[h], K[h], [t], ids, cfg.latent_rows, cfg.latent_cols, om, cfg.topk)
                ref = port.exec(q_rot[h], K[h], V[h], [t], ids, cfg.latent_rows, cfg.latent_cols, om, plan,
                                oracle.head_scale(d))
                got = att[:, h * d:(h + 1) * d]
                assert rel_l2(got, ref) <= REL_L2_TOL and max_abs(got, ref) <= MAX_ABS_TOL, (t, l, h)
            hist[l] = hist[l][-cfg.window_frames:]  # sliding eviction after the step
            # residual updates from the recorded intermediates (fp32 on the device)
            xt = rec["x"] + (rec["att"] @ w.wo).float()
            h1 = torch.nn.functional.silu((dit.rms_norm(xt, w.norm2_g) @ w.w_in).float())
            xt = xt + (h1.to(torch.bfloat16) @ w.w_out).float()
            nxt = dit.trace[l + 1]["x"] if l + 1 < len(dit.trace) else x_out
            torch.testing.assert_close(xt, nxt, rtol=0, atol=1e-5)
        assert dit.ring.frame_ids(0) == list(range(max(0, t - cfg.window_frames + 1), t + 1))
