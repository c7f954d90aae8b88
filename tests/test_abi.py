"""CPU suite: the C-ABI library loads without a GPU, exports every symbol the header
declares, validates geometry on the host exactly like the reference, and refuses to run
compute without an sm_100 device (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import pytest

import oracle
from paper_2510_12747_b200 import _abi, build
from paper_2510_12747_b200.sparse import TokenGrid, block_counts

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "fvsr_b200.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"FVSR_API\s+[\w\s\*]+?\b(fvsr_\w+)\s*\(", text)))


def test_header_declares_the_bound_symbols():
    syms = header_symbols()
    assert len(syms) >= 20
    assert syms == sorted(_abi.SIGNATURES), "SIGNATURES must mirror include/fvsr_b200.h"


def test_library_exports_every_header_symbol():
    lib = _abi.load()
    for s in header_symbols():
        assert hasattr(lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", build.LIB], capture_output=True, text=True, check=True)
    exported = {l.split()[-1] for l in out.stdout.splitlines() if " T " in l}
    assert set(header_symbols()) <= exported
    # nothing but the C-ABI is exported (-fvisibility=hidden)
    assert {s for s in exported if s.startswith("fvsr_")} == set(header_symbols())
    assert lib.fvsr_abi_version() == 1


def test_library_targets_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", build.LIB], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def test_context_requires_b200():
    """No GPU here: context creation must fail loudly, never fall back to the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = _abi.load()
    ctx = C.c_void_p()
    st = lib.fvsr_ctx_create(C.byref(ctx))
    assert st == _abi.FVSR_E_CUDA
    assert lib.fvsr_last_error()
    with pytest.raises(_abi.CudaError):
        _abi.check(st)


@pytest.mark.parametrize("qf,kf,rows,cols", [
    ([1], [0, 1], 16, 16), ([0, 1], [0, 1], 16, 16), ([5], [1, 2, 3, 4, 5], 48, 88),
    ([4, 5], [2, 3, 4, 5], 48, 88), ([3], [0, 1, 2, 3], 90, 160), ([7], [4, 5, 6, 7], 20, 28),
])
def test_block_counts_match_oracle(qf, kf, rows, cols):
    bnq, bnk = block_counts(TokenGrid(qf, rows, cols), TokenGrid(kf, rows, cols))
    assert bnq == oracle.block_count(qf, rows, cols)
    assert bnk == oracle.block_count(kf, rows, cols)


@pytest.mark.parametrize("frame_ids,rows,cols", [
    ([], 16, 16),          # TokenGrid: empty extents (P/include/vsr/grid.hpp:48-57)
    ([0], 0, 16),
    ([1, 1], 16, 16),      # strictly increasing ids
    ([2, 1], 16, 16),
    ([-1, 0], 16, 16),
])
def test_grid_validation_raises_config_error(frame_ids, rows, cols):
    with pytest.raises(_abi.ConfigError):
        block_counts(TokenGrid(frame_ids, rows, cols), TokenGrid([0], 16, 16))


def test_grids_must_share_frame_shape():
    with pytest.raises(_abi.ConfigError):
        block_counts(TokenGrid([1], 16, 16), TokenGrid([0, 1], 16, 24))


def test_error_taxonomy_matches_reference():
    """Status codes map to the reference's exception types (P/include/vsr/common.hpp:10-53)."""
    assert issubclass(_abi.ShapeError, _abi.Error)
    for code, exc in ((1, _abi.ShapeError), (2, _abi.ConfigError), (3, _abi.DegenerateRowError),
                      (4, _abi.EmptyBlockError), (5, _abi.InvariantError)):
        with pytest.raises(exc):
            _abi.check(code)
        assert oracle.ERRORS[code] == exc.__name__


def test_sparsity_csv_format_is_the_reference_one():
    """sparsity-csv-v1 header/row layout (P/src/bench.cpp:49-60; P/tests/test_config.cpp:80-87)."""
    from paper_2510_12747_b200.bench_sparsity import (SparsityRow, sparsity_csv_header, sparsity_csv_row,
                                                      topk_for_density)
    r = SparsityRow(4, 0.125, 0.1234567, 1.5, 12.0, 8.0, 0.001)
    assert sparsity_csv_header() == "k,density,flop_ratio,wall_ms_sparse,wall_ms_dense,speedup,max_abs_err_vs_dense"
    assert sparsity_csv_header().count(",") == sparsity_csv_row(r).count(",")
    assert sparsity_csv_row(r) == "4,0.125,0.123457,1.5,12,8,0.001"
    assert topk_for_density(0.136, 198) == 27 and topk_for_density(1.0, 7) == 7 and topk_for_density(0.001, 5) == 1
