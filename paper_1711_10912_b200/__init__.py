"""paper_1711_10912_b200 -- the tensorlib (TLib, arXiv:1711.10912) hot path on B200.

Drop-in for the reference's numerical core: ``ttv``, ``ttm``,
``inner_product_tensors``, ``frobenius_norm``, ``times_vectors`` and
``hopm`` over ``DenseTensor`` with runtime order, extents, one-based mode
and permutation layout.  The computation runs in hand-written sm_100a CUDA
kernels behind a C ABI (include/tensorlib_b200.h); PyTorch provides device
buffers and streams only.  There is no CPU fallback.
"""

from .contraction import (
    ContractionSpec,
    frobenius_norm,
    inner_product_flat,
    inner_product_tensors,
    outer_product,
    reduce_ttm_to_ttt,
    reduce_ttv_to_ttt,
    times_matrices,
    times_vectors,
    transpose,
    ttm,
    ttt,
    ttv,
)
from .iterators import MultiIterator, StrideIterator, fill_range, inner_product_range, walk_positions
from .hopm import DegenerateInputError, HopmRunner, HopmState, hopm, rank_one_compose, residual
from .layout import (
    MAX_INDEX,
    TensorMeta,
    compute_strides,
    first_order_layout,
    inverse_memory_index,
    last_order_layout,
    memory_index,
    volume,
    zero_indices,
)
from .tensor import DenseTensor, tensors_equal
from .views import Range, TensorView, classify_view

__version__ = "0.1.0"

__all__ = [
    "MultiIterator",
    "StrideIterator",
    "fill_range",
    "inner_product_range",
    "walk_positions",
    "Range",
    "TensorView",
    "classify_view",
    "ContractionSpec",
    "outer_product",
    "reduce_ttm_to_ttt",
    "reduce_ttv_to_ttt",
    "transpose",
    "ttt",
    "DegenerateInputError",
    "DenseTensor",
    "HopmRunner",
    "HopmState",
    "MAX_INDEX",
    "TensorMeta",
    "compute_strides",
    "first_order_layout",
    "frobenius_norm",
    "hopm",
    "inner_product_flat",
    "inner_product_tensors",
    "inverse_memory_index",
    "last_order_layout",
    "memory_index",
    "rank_one_compose",
    "residual",
    "tensors_equal",
    "times_matrices",
    "times_vectors",
    "ttm",
    "ttv",
    "volume",
    "zero_indices",
]
