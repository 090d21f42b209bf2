"""B200-native sparse polynomial multiplication (Gastineau & Laskar,
arXiv:1303.7425): a drop-in for the reference package's `mul` hot path.

Public surface mirrors the reference facade (reference __init__.py:1-55) for
the hot path: the polynomial data model, `MulConfig` and `mul`, the split
types and the cluster partition.  The product itself always runs in the CUDA
library (lib/libpolymul_b200.so); there is no CPU fallback.
"""

from .core import (SENTINEL, CoefficientOverflowError, ExponentOverflowError, Layout, Polynomial,
                   VarTable, canonicalize, check_product_fits, default_layout)
from .arrays import ArrayPolynomial
from .io import format_poly, format_text, poly_digest, text_digest, write_poly
from .parmul import MulConfig, count_below, mul, mul_arrays, native_mul
from .split import GridParams, SplitSet, select_grid
from .cluster import ClusterPlan, gpu_mul, partition_by_ops

__version__ = "0.1.0"

__all__ = [
    "SENTINEL", "CoefficientOverflowError", "ExponentOverflowError", "Layout", "Polynomial",
    "VarTable", "canonicalize", "check_product_fits", "default_layout", "format_poly",
    "poly_digest", "ArrayPolynomial", "format_text", "text_digest", "write_poly", "MulConfig",
    "count_below", "mul", "mul_arrays", "native_mul", "GridParams", "SplitSet",
    "select_grid", "ClusterPlan", "gpu_mul", "partition_by_ops", "__version__",
]
