"""paper_2508_11385_b200 — B200-native fused element-wise expression + reduction
engine (the data-parallel hot path of Bandicoot, arXiv 2508.11385).

The compute path is libcoot.so (hand-written CUDA for sm_100a behind the C ABI
of include/coot.h); this package is its thin Python binding plus the
delayed-evaluation expression builder.  Importing it fails loudly if the
native library is missing — there is no CPU fallback.
"""
from . import _native  # noqa: F401  (raises ImportError if libcoot.so is missing)
from ._native import CootError
from .api import (Col, Context, Expr, Mat, Row, View, abs, accu, default_ctx, dot, exp,
                  index_max, index_min, init, log, lower, max, mean, min, minmax, norm2,
                  partial_bytes, shard_range, sqrt, square, stddev, sum, validate, var)

__all__ = ["Col", "Context", "CootError", "Expr", "Mat", "Row", "View", "abs", "accu",
           "default_ctx", "dot", "exp", "index_max", "index_min", "init", "log", "lower", "max",
           "mean", "min", "minmax", "norm2", "partial_bytes", "shard_range", "sqrt", "square",
           "stddev", "sum", "validate", "var"]
