"""B200-native sparse polynomial multiplication (Gastineau & Laskar,
arXiv:1303.7425): a drop-in for the reference package's `mul` hot path.

Public surface mirrors the reference facade (reference __init__.py:1-55) for
the hot path: the polynomial data model, `MulConfig` and `mul`, the split
types and the cluster partition.  The product itself always runs in the CUDA
library (lib/libpolymul_b200.so); there is no CPU fallback.
"""

from .core import (SENTINEL, CoefficientOverflowError, ExponentOverflowError, Layout, Polynomial,
                   VarTable, canonicalize, check_product_fits, default_layout, naive_mul)
from .arrays import ArrayPolynomial
from .io import (PolyIOError, format_poly, format_text, parse_poly, poly_digest, read_poly, text_digest,
                 write_poly)
from .expr import ExprSyntaxError, poly_from_expr
from .expr import evaluate as eval_expr
from .expr import parse as parse_expr
from .parmul import MulConfig, count_below, mul, mul_arrays, native_mul
from .split import GridParams, SplitSet, select_grid
from .cluster import ClusterPlan, gpu_mul, partition_by_ops

__version__ = "0.1.0"

__all__ = [
    "SENTINEL", "CoefficientOverflowError", "ExponentOverflowError", "Layout", "Polynomial",
    "VarTable", "canonicalize", "check_product_fits", "default_layout", "naive_mul", "format_poly",
    "PolyIOError", "parse_poly", "read_poly", "ExprSyntaxError", "poly_from_expr", "eval_expr",
    "parse_expr",
    "poly_digest", "ArrayPolynomial", "format_text", "text_digest", "write_poly", "MulConfig",
    "count_below", "mul", "mul_arrays", "native_mul", "GridParams", "SplitSet",
    "select_grid", "ClusterPlan", "gpu_mul", "partition_by_ops", "__version__",
]
