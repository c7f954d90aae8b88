"""sparsity-csv-v1 on the GPU (P/src/bench.cpp:49-114): same header and row
format as the reference; density and flop_ratio columns identical to the reference-pinned
oracle's sparsity_report of the same (bit-exact) plans; the sparse outputs converge to the
dense baseline as k grows (exactly equal at k = bnk)."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

fv = pytest.importorskip("paper_2510_12747_b200")
from paper_2510_12747_b200.bench_sparsity import (BenchConfig, bench_sparsity, sparsity_csv_header,  # noqa: E402
                                                  sparsity_csv_row)


def test_sparsity_csv_matches_reference_accounting():
    cfg = BenchConfig(frames=4, rows=32, cols=64, d_head=64, reps=3)
    frames = list(range(cfg.frames))
    L = cfg.frames * cfg.rows * cfg.cols
    port = oracle.Port()
    q, k, v = (oracle.bf16_round(port.gaussian(4200 + i, L * cfg.d_head).reshape(L, cfg.d_head)) for i in range(3))
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda().to(torch.bfloat16)
    sweep = [1, 2, 4, 8, 16, 32, 64]
    rows = bench_sparsity(cfg, sweep, dev(q), dev(k), dev(v))
    assert sparsity_csv_header() == "k,density,flop_ratio,wall_ms_sparse,wall_ms_dense,speedup,max_abs_err_vs_dense"
    bnk = oracle.block_count(frames, cfg.rows, cfg.cols)
    for r in rows:
        line = sparsity_csv_row(r)
        assert line.count(",") == sparsity_csv_header().count(",")
        assert line.startswith(f"{r.k},")
        plan = port.plan(q, k, frames, frames, cfg.rows, cfg.cols, oracle.Mask.all(), r.k)
        rep = port.report(frames, frames, cfg.rows, cfg.cols, oracle.Mask.all(), plan, L)
        assert line.split(",")[1] == "%.6g" % rep["density"], (r.k, line, rep)
        assert line.split(",")[2] == "%.6g" % (rep["executed_pairs"] / rep["dense_pairs"]), (r.k, line, rep)
        assert r.wall_ms_sparse > 0 and r.wall_ms_dense > 0
        if r.k >= bnk:
            assert r.max_abs_err_vs_dense == 0.0
    assert rows[-1].max_abs_err_vs_dense <= rows[0].max_abs_err_vs_dense
