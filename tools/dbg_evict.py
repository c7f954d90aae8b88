"""Repro helper: the scored-eviction ring loop with a synchronize after every call."""
import numpy as np
import torch
import paper_2510_12747_b200 as fv
import oracle

ctx = fv.Context.default()
ctx.set_flags(1)
heads, rows, cols, d, topk, window = 2, 16, 40, 128, 4, 3
n = rows * cols
ring = fv.KVRing(1, heads, d, rows, cols, window)
port = oracle.Port()
for t in range(10):
    x = oracle.bf16_round(np.stack([port.gaussian(800 + 10 * t + h, 3 * n * d).reshape(3, n, d) for h in range(heads)]))
    q, k, v = [torch.from_numpy(np.ascontiguousarray(x[:, i])).to("cuda", torch.bfloat16) for i in range(3)]
    ring.append(0, t, k, v)
    torch.cuda.synchronize()
    print("append ok", t, flush=True)
    out = ring.attention(0, q, [t], fv.Mask.all_allowed(), topk)
    torch.cuda.synchronize()
    print("attention ok", t, flush=True)
    mass = ring.frame_mass(0, [t], fv.Mask.all_allowed()).cpu().numpy()
    torch.cuda.synchronize()
    print("mass ok", t, flush=True)
    ring.evict_scored(0, 1, mass)
