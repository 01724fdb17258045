"""B200-native adaptive fp64 CSR SpMV (arXiv 1711.05487 hot path).

Thin Python binding over ``libspmv.so`` (C ABI declared in
``include/spmv.h``). Argument marshalling only: every step of the path
(upload, inspector, selection, structure build, SpMV, iterated mode) runs in
the native library and its sm_100a kernels. There is no CPU fallback: if the
library is missing this package fails to import.
"""
from .binding import (  # noqa: F401
    ARR, VARIANTS, CLASSES, Options, Plan, SpmvError, device_query, kernel_launches, lib, norm_partial_count,
    select, shard_bounds,
)

__all__ = ["Plan", "Options", "SpmvError", "shard_bounds", "select", "device_query", "kernel_launches",
           "norm_partial_count", "ARR", "VARIANTS", "CLASSES", "lib"]
