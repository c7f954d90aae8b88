"""B200-native FlashVSR locality-constrained block-sparse streaming attention.

Hot path of arXiv 2510.12747's streaming DiT, rebuilt for sm_100a behind the reference's
operator API (P/include/vsr/sparse.hpp, P/include/vsr/kv_cache.hpp; P =
/root/reference/proj).  The compute lives in libfvsr_b200.so (C-ABI:
include/fvsr_b200.h); this package is the thin Python mirror used by tests and benches.
"""
from ._abi import (ConfigError, CudaError, DegenerateRowError, EmptyBlockError, Error, InvariantError,
                   ShapeError)
from .kv_ring import EVICT_HEAD_WISE, EVICT_SLIDING, EVICT_UNIFORM, KVRing
from .sparse import (Context, Mask, SparsePlan, SparsityReport, TokenGrid, block_counts, build_causal_mask,
                     build_segment_mask, frame_attention_mass,
                     plan_sparse, sparse_attention_exec, sparsity_report)

__all__ = [
    "ConfigError", "CudaError", "DegenerateRowError", "EmptyBlockError", "Error", "InvariantError", "ShapeError",
    "Context", "KVRing", "Mask", "SparsePlan", "SparsityReport", "TokenGrid", "block_counts", "plan_sparse",
    "sparse_attention_exec", "sparsity_report", "frame_attention_mass", "EVICT_SLIDING", "EVICT_UNIFORM",
    "EVICT_HEAD_WISE", "build_segment_mask", "build_causal_mask",
]
