"""Head-parallel sharding of the streaming attention layer-step over N GPUs of one node.

The reference processes heads serially (P/src/stream.cpp:237-256; P =
/root/reference/proj); heads and, within a head, query tiles are independent given K/V,
so the (head, q-tile) work units shard with no exchange except gathering the outputs.

    units  = heads * n_trows * tiles       (unit = head*(n_trows*tiles) + trow*tiles + tile)
             a temporal row holds one query frame (64 rows per unit) or the two frames
             2m, 2m+1 of a (2,8,8) q-block (128 rows per unit, the Tq=2 chunk): unit_space()
    rank r owns units [r*per, min(U, (r+1)*per)), per = ceil(U / N)
    ring   = KV for heads [h0, h1) that its units touch (a head split across two ranks
             has its K/V on both; 12 heads over 8 GPUs split 1.5 heads per rank)
    output = tile-major shard [per, 64, d]  ->  NCCL all_gather_into_tensor (equal chunks)
             -> untile() back to [heads, Lq, d] token order when a consumer needs it.

Uniform scored eviction (KVCache::evict, P/src/kv_cache.cpp:118-128) sums frame scores over
ALL heads, but a rank's ring holds only heads [h0, h1).  full_frame_mass() is the one extra
exchange: each rank writes its heads' rows into a [heads, frames] float64 matrix (zeros
elsewhere) and an all-reduce(MAX) assembles it (masses are >= 0; a head held by two ranks has
identical rows on both, so MAX takes it once).  uniform_evict() then applies the global
decision to the local ring: every rank evicts the same frames.

The gather of layer l runs on NCCL's stream while layer l+1 computes (async_op, double
buffered); the step's host code never waits on it until the buffer is reused.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Tuple

import torch


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    total_units: int
    per: int          # units per rank (padded)
    u0: int           # first unit owned
    u1: int           # one past the last unit owned
    units_per_head: int
    h0: int           # first head touched
    h1: int           # one past the last head touched

    @property
    def local_unit_begin(self) -> int:
        return self.u0 - self.h0 * self.units_per_head

    @property
    def local_unit_end(self) -> int:
        return self.u1 - self.h0 * self.units_per_head

    @property
    def heads(self) -> int:
        return self.h1 - self.h0


def unit_space(q_frame_ids) -> Tuple[int, int]:
    """(n_trows, frames_per_unit) of the attention kernel's unit space for these query frames:
    consecutive frames sharing frame // 2 form one temporal row (P/src/partition.cpp:38-62).
    Sharded (unit-range / tile-major) attention needs rows of equal height."""
    ids = [int(f) for f in q_frame_ids]
    counts = []
    for i, f in enumerate(ids):
        if i > 0 and f // 2 == ids[i - 1] // 2:
            counts[-1] += 1
        else:
            counts.append(1)
    if len(set(counts)) != 1:
        raise ValueError("head-parallel attention needs query temporal rows of equal height "
                         f"(frames {ids} give rows of {counts} frames)")
    return len(counts), counts[0]


def shard(total_units: int, units_per_head: int, world: int, rank: int) -> Shard:
    per = -(-total_units // world)
    u0 = min(total_units, rank * per)
    u1 = min(total_units, u0 + per)
    if u1 > u0:
        h0, h1 = u0 // units_per_head, (u1 - 1) // units_per_head + 1
    else:
        h0 = h1 = 0
    return Shard(rank, world, total_units, per, u0, u1, units_per_head, h0, h1)


def untile_index(heads: int, nq: int, rows: int, cols: int, device=None,
                 frames_per_unit: int = 1) -> Tuple[torch.Tensor, torch.Tensor]:
    """(src_row, dst_row) index pairs mapping tile-major rows [units * 64*frames_per_unit]
    to token-major rows [heads*nq*rows*cols]; padding rows of ragged tiles are dropped.
    frames_per_unit = 2 for paired query frames (unit_space), whose units hold 128 rows:
    rows 0-63 frame 2m, rows 64-127 frame 2m+1 of the same 8x8 tile."""
    tw, th = (cols + 7) // 8, (rows + 7) // 8
    tiles = tw * th
    fpu = int(frames_per_unit)
    if nq % fpu:
        raise ValueError("nq must be a multiple of frames_per_unit")
    ntr = nq // fpu
    u = torch.arange(heads * ntr * tiles, device=device)
    r = torch.arange(64 * fpu, device=device)
    head = (u // (ntr * tiles))[:, None]
    f = ((u % (ntr * tiles)) // tiles)[:, None] * fpu + r[None, :] // 64
    tile = (u % tiles)[:, None]
    rr = r[None, :] % 64
    h = (tile // tw) * 8 + rr // 8
    w = (tile % tw) * 8 + rr % 8
    valid = (h < rows) & (w < cols)
    dst = (head * nq + f) * rows * cols + h * cols + w
    src = u[:, None] * (64 * fpu) + r[None, :]
    return src[valid], dst[valid]


def untile(tiles: torch.Tensor, heads: int, nq: int, rows: int, cols: int, index=None,
           frames_per_unit: int = 1) -> torch.Tensor:
    """Tile-major [>=units, 64*frames_per_unit, d] -> token-major [heads, nq*rows*cols, d]."""
    d = tiles.shape[-1]
    src, dst = index if index is not None else untile_index(heads, nq, rows, cols, tiles.device, frames_per_unit)
    out = torch.empty((heads * nq * rows * cols, d), dtype=tiles.dtype, device=tiles.device)
    out[dst] = tiles.reshape(-1, d)[src]
    return out.view(heads, nq * rows * cols, d)


class Gatherer:
    """Double-buffered async all-gather of tile-major shards (torch.distributed, NCCL/gloo)."""

    def __init__(self, sh: Shard, d: int, device, dtype=torch.bfloat16, group=None, frames_per_unit: int = 1):
        self.sh, self.group = sh, group
        rows = 64 * int(frames_per_unit)
        self.shards = [torch.zeros((sh.per, rows, d), dtype=dtype, device=device) for _ in range(2)]
        self.full = [torch.empty((sh.per * sh.world, rows, d), dtype=dtype, device=device) for _ in range(2)]
        self.work = [None, None]
        self.i = 0

    def next_shard(self) -> torch.Tensor:
        """Shard buffer for the next layer-step; waits for the gather that last used it."""
        self.i ^= 1
        if self.work[self.i] is not None:
            self.work[self.i].wait()
            self.work[self.i] = None
        return self.shards[self.i]

    def launch(self) -> None:
        import torch.distributed as dist
        self.work[self.i] = dist.all_gather_into_tensor(self.full[self.i], self.shards[self.i], group=self.group,
                                                        async_op=True)

    def result(self) -> torch.Tensor:
        if self.work[self.i] is not None:
            self.work[self.i].wait()
            self.work[self.i] = None
        return self.full[self.i][: self.sh.total_units]

    def drain(self) -> None:
        for i in range(2):
            if self.work[i] is not None:
                self.work[i].wait()
                self.work[i] = None


def full_frame_mass(local: torch.Tensor, sh: Shard, heads_total: int, group=None) -> torch.Tensor:
    """[heads_total, frames] float64 frame masses on every rank from each rank's
    [sh.heads, frames] rows (KVRing.frame_mass of its ring)."""
    import torch.distributed as dist
    full = torch.zeros((heads_total, local.shape[1]), dtype=torch.float64, device=local.device)
    if sh.heads:
        full[sh.h0:sh.h1] = local.to(torch.float64)
    if dist.is_initialized() and sh.world > 1:
        dist.all_reduce(full, op=dist.ReduceOp.MAX, group=group)
    return full


def uniform_total(full: torch.Tensor):
    """Per-frame sum over heads in head order, in double (kv_cache.cpp:123-125)."""
    rows = full.detach().cpu().tolist()
    total = [0.0] * len(rows[0])
    for r in rows:
        for i, x in enumerate(r):
            total[i] += x
    return total


def uniform_evict(ring, layer: int, full: torch.Tensor) -> None:
    """KVCache::evict(uniform) with the GLOBAL head sum applied to this rank's ring: the total
    goes in row 0 and the other rows are zero, so the ring's own head sum reproduces it exactly."""
    from .kv_ring import EVICT_UNIFORM
    total = uniform_total(full)
    scores = torch.zeros((ring.heads, len(total)), dtype=torch.float64)
    scores[0] = torch.tensor(total, dtype=torch.float64)
    ring.evict_scored(layer, EVICT_UNIFORM, scores)
