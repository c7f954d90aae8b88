"""bench_sparsity on the GPU: the reference's sparsity sweep (P/src/bench.cpp:71-114,
P = /root/reference/proj) through this package's operators, emitting the same
sparsity-csv-v1 rows (header and %.6g formatting of P/src/bench.cpp:49-60).

    rows = bench_sparsity(BenchConfig(frames=4, rows=32, cols=64, d_head=64), [1, 2, 4, 8])
    print(sparsity_csv_header()); [print(sparsity_csv_row(r)) for r in rows]

Like the reference: self attention over a TokenGrid of `frames` frames, all-allowed mask,
q/k/v ~ N(0,1) (here torch's generator, rounded to bf16), plan_sparse + sparsity_report +
sparse_attention_exec per k, and a dense baseline.  Differences, stated:
  * wall_ms_* are CUDA-event medians of the device kernels (plan excluded, as in the
    reference, which times only sparse_attention_exec);
  * the dense baseline (wall_ms_dense, the reference's dense_attention_stream) is the same
    tensor-core kernel with every allowed block selected (k = bnk): exact dense attention;
  * d_head must be 64 or 128 (the tensor-core kernel's head dims; the reference default 32
    is not supported).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Sequence

import torch

from .sparse import Mask, TokenGrid, block_counts, plan_sparse, sparse_attention_exec, sparsity_report


@dataclass
class BenchConfig:
    """The [grid] / [attention] / [bench] knobs bench_sparsity reads (P/include/vsr/config.hpp:47-80)."""
    frames: int = 4
    rows: int = 32
    cols: int = 64
    d_head: int = 64
    seed: int = 42
    reps: int = 5
    warmup: int = 1

    def validate(self) -> None:
        from ._abi import ConfigError
        if self.frames < 1 or self.rows < 1 or self.cols < 1:
            raise ConfigError("bench config: empty grid")
        if self.d_head not in (64, 128):
            raise ConfigError("bench_sparsity (GPU): d_head must be 64 or 128")
        if self.reps < 1:
            raise ConfigError("bench config: reps must be >= 1")


@dataclass
class SparsityRow:
    """vsr::SparsityRow (P/include/vsr/bench.hpp)."""
    k: int
    density: float
    flop_ratio: float
    wall_ms_sparse: float
    wall_ms_dense: float
    speedup: float
    max_abs_err_vs_dense: float


def _fmt(v: float) -> str:  # std::snprintf("%.6g")
    return "%.6g" % v


def sparsity_csv_header() -> str:
    return "k,density,flop_ratio,wall_ms_sparse,wall_ms_dense,speedup,max_abs_err_vs_dense"


def sparsity_csv_row(r: SparsityRow) -> str:
    return ",".join([str(int(r.k)), _fmt(r.density), _fmt(r.flop_ratio), _fmt(r.wall_ms_sparse),
                     _fmt(r.wall_ms_dense), _fmt(r.speedup), _fmt(r.max_abs_err_vs_dense)])


def topk_for_density(target_density: float, key_blocks: int) -> int:
    """P/src/bench.cpp:62-69."""
    import math
    from ._abi import ConfigError
    if not (0.0 < target_density <= 1.0):
        raise ConfigError("topk_for_density: target must be in (0, 1]")
    if key_blocks <= 0:
        raise ConfigError("topk_for_density: no key blocks")
    return max(1, int(math.ceil(target_density * key_blocks - 1e-9)))


def _median_ms(fn, reps: int, warmup: int) -> float:
    for _ in range(warmup):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    n = len(ts)
    return ts[n // 2] if n % 2 else 0.5 * (ts[n // 2 - 1] + ts[n // 2])


def bench_sparsity(cfg: BenchConfig, k_sweep: Sequence[int], q=None, k=None, v=None) -> List[SparsityRow]:
    """P/src/bench.cpp:71-114 on the device; q/k/v [L, d] bf16 CUDA tensors may be given."""
    from ._abi import ConfigError
    cfg.validate()
    if not k_sweep:
        raise ConfigError("bench_sparsity: empty k sweep")
    grid = TokenGrid(cfg.frames, cfg.rows, cfg.cols)
    L = grid.token_count()
    if q is None:
        gen = torch.Generator(device="cuda").manual_seed(cfg.seed)
        q, k, v = (torch.randn((L, cfg.d_head), generator=gen, device="cuda").to(torch.bfloat16) for _ in range(3))
    mask = Mask.all_allowed()
    scale = 1.0 / float(cfg.d_head) ** 0.5
    _, bnk = block_counts(grid, grid)
    dense_plan = plan_sparse(q, k, grid, grid, mask, bnk)
    dense = sparse_attention_exec(q, k, v, dense_plan, mask, scale)
    dense_ms = _median_ms(lambda: sparse_attention_exec(q, k, v, dense_plan, mask, scale, out=dense,
                                                        check_errors=False), cfg.reps, cfg.warmup)
    rows = []
    for kk in k_sweep:
        plan = plan_sparse(q, k, grid, grid, mask, int(kk))
        rep = sparsity_report(plan, mask)
        out = sparse_attention_exec(q, k, v, plan, mask, scale)
        sparse_ms = _median_ms(lambda: sparse_attention_exec(q, k, v, plan, mask, scale, out=out, check_errors=False),
                               cfg.reps, cfg.warmup)
        err = float((out.float() - dense.float()).abs().max())
        rows.append(SparsityRow(int(kk), rep.density, rep.flop_ratio, sparse_ms, dense_ms,
                                dense_ms / sparse_ms if sparse_ms > 0 else 0.0, err))
    return rows
