"""CPU suite: head-parallel sharding — shard arithmetic, tile-major <->
token-major layout, and the all-gather path at world size 2 over gloo."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_12747_b200.head_parallel import (Gatherer, full_frame_mass, shard, uniform_total, unit_space, untile,
                                                 untile_index)


@pytest.mark.parametrize("heads,nq,tiles,world", [(12, 1, 66, 1), (12, 1, 66, 2), (12, 1, 66, 4),
                                                  (12, 1, 66, 8), (12, 2, 66, 8), (5, 1, 7, 3),
                                                  (1, 1, 4, 8)])
def test_shards_partition_units(heads, nq, tiles, world):
    uph = nq * tiles
    total = heads * uph
    seen = []
    for r in range(world):
        s = shard(total, uph, world, r)
        assert s.u1 - s.u0 <= s.per
        seen.extend(range(s.u0, s.u1))
        if s.u1 > s.u0:
            assert s.h0 * uph <= s.u0 and s.u1 <= s.h1 * uph   # its KV heads cover its units
            assert 0 <= s.local_unit_begin < s.local_unit_end <= s.heads * uph
    assert seen == list(range(total))


@pytest.mark.parametrize("rows,cols,nq", [(16, 16, 1), (20, 28, 1), (48, 88, 2), (13, 9, 1)])
def test_untile_inverts_tiling(rows, cols, nq):
    heads, d = 3, 4
    x = torch.randn(heads, nq * rows * cols, d)
    tw, th = (cols + 7) // 8, (rows + 7) // 8
    # build the tile-major layout directly (ring attention's FVSR_OUT_TILE_MAJOR)
    tiles = torch.zeros(heads * nq * tw * th, 64, d)
    for h in range(heads):
        for f in range(nq):
            for t in range(tw * th):
                for r in range(64):
                    hh, ww = (t // tw) * 8 + r // 8, (t % tw) * 8 + r % 8
                    if hh < rows and ww < cols:
                        tiles[(h * nq + f) * tw * th + t, r] = x[h, f * rows * cols + hh * cols + ww]
    assert torch.equal(untile(tiles, heads, nq, rows, cols), x)
    src, dst = untile_index(heads, nq, rows, cols)
    assert dst.numel() == heads * nq * rows * cols and torch.equal(dst.sort().values, torch.arange(dst.numel()))


@pytest.mark.parametrize("rows,cols", [(16, 16), (20, 28), (13, 9)])
def test_untile_paired_query_frames(rows, cols):
    """Paired query frames (2m, 2m+1: one temporal row, the Tq=2 chunk): the kernel's unit is
    [128 rows] = frame 2m tile rows 0-63 then frame 2m+1 (kernel_attn.cu NQ=128)."""
    heads, d, qf = 2, 4, [6, 7]
    ntr, fpu = unit_space(qf)
    assert (ntr, fpu) == (1, 2)
    nq = len(qf)
    x = torch.randn(heads, nq * rows * cols, d)
    tw, th = (cols + 7) // 8, (rows + 7) // 8
    tiles = torch.zeros(heads * ntr * tw * th, 128, d)
    for h in range(heads):
        for t in range(tw * th):
            for r in range(128):
                f, rr = r // 64, r % 64
                hh, ww = (t // tw) * 8 + rr // 8, (t % tw) * 8 + rr % 8
                if hh < rows and ww < cols:
                    tiles[h * tw * th + t, r] = x[h, f * rows * cols + hh * cols + ww]
    assert torch.equal(untile(tiles, heads, nq, rows, cols, frames_per_unit=2), x)
    assert unit_space([5, 6]) == (2, 1) and unit_space([4, 5, 6, 7]) == (2, 2)
    with pytest.raises(ValueError):
        unit_space([3, 4, 5])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, heads, nq, rows, cols, d, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        tw, th = (cols + 7) // 8, (rows + 7) // 8
        uph = nq * tw * th
        total = heads * uph
        torch.manual_seed(0)
        full = torch.randn(total, 64, d)          # what one GPU would compute, tile-major
        sh = shard(total, uph, world, rank)
        g = Gatherer(sh, d, "cpu", dtype=torch.float32)
        outs = []
        for step in range(3):                       # double-buffered, gathers in flight
            buf = g.next_shard()
            buf.zero_()
            buf[: sh.u1 - sh.u0] = full[sh.u0:sh.u1] + step
            g.launch()
            outs.append((step, g))
            res = g.result()
            ok = torch.equal(res, full + step)
            tok = untile(res, heads, nq, rows, cols)
            ok = ok and torch.equal(tok, untile(full + step, heads, nq, rows, cols))
            if not ok:
                q.put((rank, "mismatch", step))
                return
        g.drain()
        q.put((rank, "ok", None))
        dist.destroy_process_group()
    except Exception as e:  # surface to the parent
        q.put((rank, "error", repr(e)))


@pytest.mark.parametrize("heads,rows,cols,nq", [(12, 48, 88, 1), (3, 20, 28, 1), (2, 16, 16, 2)])
def test_gather_world2_gloo(heads, rows, cols, nq):
    world, d = 2, 8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, heads, nq, rows, cols, d, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] == "ok" for r in results), results


def _mass_worker(rank, world, port, heads, uph, n, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.manual_seed(1)
        full = torch.rand(heads, n, dtype=torch.float64)  # what one GPU's ring would report
        sh = shard(heads * uph, uph, world, rank)
        got = full_frame_mass(full[sh.h0:sh.h1].clone(), sh, heads)
        q.put((rank, "ok" if torch.equal(got, full) else "mismatch", uniform_total(got)))
        dist.destroy_process_group()
    except Exception as e:
        q.put((rank, "error", repr(e)))


@pytest.mark.parametrize("heads,uph", [(12, 66), (3, 5)])  # (3, 5): head 1 is split across the two ranks
def test_uniform_eviction_scores_world2_gloo(heads, uph):
    """Uniform eviction under head-parallel sharding (kv_cache.cpp:118-128): the all-reduce
    rebuilds every head's frame masses on every rank, so all ranks take the same decision,
    equal to the single-process one (oracle.evict)."""
    import numpy as np
    import oracle
    world, n = 2, 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mass_worker, args=(r, world, port, heads, uph, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] == "ok" for r in results), results
    assert results[0][2] == results[1][2]
    torch.manual_seed(1)
    full = torch.rand(heads, n, dtype=torch.float64).numpy()
    ids = [3, 4, 5, 6, 7]
    want = oracle.evict(1, 3, ids, full, heads)[0]
    total = results[0][2]
    got = [i for i in ids if i not in oracle.evict_victims(ids, total, len(ids) - 3)]
    assert got == want
