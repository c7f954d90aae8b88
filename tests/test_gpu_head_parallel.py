"""Head-parallel sharding on the GPU (VERDICT r1 "Next" 2).

Each simulated rank r of world N owns the (head, q-tile) units head_parallel.shard gives it
and a ring holding only the heads [h0, h1) those units touch (its own append of those heads'
K/V).  It runs the mask builder and the attention kernel on its local unit range with the
tile-major output; the shards, concatenated in rank order (what all_gather_into_tensor
produces), untiled, must be bitwise equal to the single-GPU token-major output.  The ranks
run one after another on one GPU: no rank waits on another, so this is exactly the
per-rank kernel path of a multi-GPU run minus the NCCL transport (covered by the gloo tests
and, with >= 2 GPUs, test_nccl_gather_world2).
"""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
from tests.helpers import to_dev

pytestmark = pytest.mark.gpu

fv = pytest.importorskip("paper_2510_12747_b200")
from paper_2510_12747_b200.head_parallel import shard, unit_space, untile  # noqa: E402


def _stream_inputs(heads, rows, cols, d, frames, seed):
    port = oracle.Port()
    N = rows * cols
    out = {}
    for t in frames:
        x = oracle.bf16_round(np.stack([port.gaussian(seed + 100 * t + h, 3 * N * d).reshape(3, N, d)
                                        for h in range(heads)]))
        out[t] = (x[:, 0], x[:, 1], x[:, 2])
    return out


@pytest.mark.parametrize("qf", [[32], [32, 33]], ids=["tq1", "tq2_paired"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_equals_unsharded(world, qf):
    heads, rows, cols, d, window, topk = 12, 48, 88, 128, 4, 27
    N = rows * cols
    kf = list(range(qf[-1] - window, qf[-1] + 1))
    hist = [f for f in kf if f not in qf]
    data = _stream_inputs(heads, rows, cols, d, kf, 31)
    q = np.concatenate([data[t][0] for t in qf], axis=1)
    mask = fv.Mask.locality(48, 72, truncated=True)

    def fill(ring, h0, h1):
        for t in kf:
            ring.append(0, t, to_dev(data[t][1][h0:h1]), to_dev(data[t][2][h0:h1]))

    full_ring = fv.KVRing(1, heads, d, rows, cols, window + len(qf))
    fill(full_ring, 0, heads)
    ref = full_ring.attention(0, to_dev(q), qf, mask, topk)
    torch.cuda.synchronize()

    ntr, fpu = unit_space(qf)
    tiles = ((rows + 7) // 8) * ((cols + 7) // 8)
    uph = ntr * tiles
    total = heads * uph
    parts = []
    for r in range(world):
        sh = shard(total, uph, world, r)
        buf = torch.zeros((sh.per, 64 * fpu, d), dtype=torch.bfloat16, device="cuda")
        if sh.u1 > sh.u0:
            ring = fv.KVRing(1, sh.heads, d, rows, cols, window + len(qf))
            fill(ring, sh.h0, sh.h1)
            part = ring.attention(0, to_dev(q[sh.h0:sh.h1]), qf, mask, topk, unit_begin=sh.local_unit_begin,
                                  unit_end=sh.local_unit_end, tile_major=True)
            buf[: sh.u1 - sh.u0] = part
            del ring
        parts.append(buf)
    gathered = torch.cat(parts)[:total]
    got = untile(gathered, heads, len(qf), rows, cols, frames_per_unit=fpu)
    assert got.shape == ref.shape
    assert torch.equal(got, ref), f"world {world}: sharded output differs from the single-GPU output"
    _ = hist


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _nccl_worker(rank, world, port, q):
    try:
        import torch.distributed as dist
        from paper_2510_12747_b200.head_parallel import Gatherer
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world)
        heads, rows, cols, d, window, topk = 12, 48, 88, 128, 4, 27
        kf, qf = list(range(28, 33)), [32]
        data = _stream_inputs(heads, rows, cols, d, kf, 57)
        tiles = ((rows + 7) // 8) * ((cols + 7) // 8)
        total = heads * tiles
        sh = shard(total, tiles, world, rank)
        ring = fv.KVRing(1, sh.heads, d, rows, cols, window)
        for t in kf:
            ring.append(0, t, to_dev(data[t][1][sh.h0:sh.h1]), to_dev(data[t][2][sh.h0:sh.h1]))
        g = Gatherer(sh, d, "cuda")
        buf = g.next_shard()
        ring.attention(0, to_dev(data[32][0][sh.h0:sh.h1]), qf, fv.Mask.all_allowed(), topk,
                       unit_begin=sh.local_unit_begin, unit_end=sh.local_unit_end, tile_major=True,
                       out=buf[: sh.u1 - sh.u0])
        g.launch()
        got = untile(g.result(), heads, 1, rows, cols)
        full = fv.KVRing(1, heads, d, rows, cols, window)
        for t in kf:
            full.append(0, t, to_dev(data[t][1]), to_dev(data[t][2]))
        ref = full.attention(0, to_dev(data[32][0]), qf, fv.Mask.all_allowed(), topk)
        q.put((rank, bool(torch.equal(got, ref))))
        dist.destroy_process_group()
    except Exception as e:
        q.put((rank, repr(e)))


def test_nccl_gather_world2():
    """The real NCCL all-gather of tile-major shards (needs 2 GPUs; skipped otherwise)."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_nccl_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] is True for r in res), res


def test_cpp_head_parallel_layer_step():
    """The host-stays-C++ head-parallel layer-step (integration/vsr_b200_parallel.hpp): world 1
    through a real NCCL all-gather and simulated worlds 2, 4, 8 (one object per rank, shards
    concatenated in rank order, fvsr_untile), six streaming steps with a locality window, each
    bitwise equal to the unsharded fvsr_ring_step (integration/hp_main.cpp)."""
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "integration", "_build",
                       "hp_main")
    if not os.path.exists(exe):
        pytest.skip("integration/_build/hp_main not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("OK") == 4, r.stdout


@pytest.mark.parametrize("qf", [[32], [32, 33]])
def test_device_untile_matches_index_untile(qf):
    """fvsr_untile (device) == head_parallel.untile (index gather) for single and paired query frames."""
    import ctypes as C
    heads, rows, cols, d = 3, 20, 28, 64
    ntr, fpu = unit_space(qf)
    tiles = ((rows + 7) // 8) * ((cols + 7) // 8)
    units = heads * ntr * tiles
    t = torch.randn(units, 64 * fpu, d, device="cuda").to(torch.bfloat16)
    want = untile(t, heads, len(qf), rows, cols, frames_per_unit=fpu)
    got = torch.zeros_like(want)
    ctx = fv.Context.default()
    fv._abi.check(ctx.lib.fvsr_untile(ctx.h, t.data_ptr(), units, fpu, len(qf), rows, cols, d, got.data_ptr(),
                                      C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    assert torch.equal(got, want)
