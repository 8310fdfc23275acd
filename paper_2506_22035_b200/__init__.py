"""B200-native SPIDER stencil engine (arXiv 2506.22035), drop-in for the
reference `sparsestencil` hot path.

A stencil is lowered to a GEMM per kernel row; the AOT strided column swap
makes each kernel-row matrix 2:4 structured-sparse, the matching input rows are
permuted on the fly while the B operand is staged, and the product runs on
Blackwell sparse tensor cores (tcgen05.mma.sp, sm_100a).  The names below
mirror the reference package's public API for stencil definition, transform
and apply (reference __init__.py:9-88); the device engine, the 3D extension
and the multi-GPU slab driver are additions.
"""
from .core import (
    Grid,
    Grid3D,
    Shape,
    StencilKernel,
    grid_from_interior,
    make_kernel,
    make_kernel_3d,
    random_grid,
    random_grid_3d,
)
from .transform import (
    Check24Report,
    CompressedKernel,
    KernelMatrix,
    Parity,
    RowPermutation,
    band_rows,
    build_kernel_matrix,
    check_2to4,
    decode,
    encode,
    encode_segment,
    input_row_permutation,
    metadata_from_bytes,
    metadata_to_bytes,
    sparsity_ratio,
    sptc_compatible,
    strided_swap,
    swap_columns,
)

from .io import load_grid, load_kernel, save_grid, save_kernel

__version__ = "0.1.0"


_LAZY_PIPELINE = {"ExecConfig", "DeviceConfig", "ExecStats", "TransformedStencil", "transform_stencil", "execute",
                  "naive_apply", "verify", "report_json", "max_rel_error", "get_plan", "DEFAULT_TOLERANCE"}
_LAZY_ENGINE = {"Plan", "DeviceGrid", "naive_apply_device", "mma_selftest"}


def __getattr__(name):
    # The execution layer imports torch; load it lazily so the transform layer
    # stays importable (and cheap) on its own.
    import importlib

    if name in _LAZY_PIPELINE:
        return getattr(importlib.import_module(".pipeline", __name__), name)
    if name in _LAZY_ENGINE:
        return getattr(importlib.import_module(".engine", __name__), name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")


__all__ = [
    "load_grid",
    "load_kernel",
    "save_grid",
    "save_kernel",
    "Grid",
    "Grid3D",
    "Shape",
    "StencilKernel",
    "grid_from_interior",
    "make_kernel",
    "make_kernel_3d",
    "random_grid",
    "random_grid_3d",
    "Check24Report",
    "CompressedKernel",
    "KernelMatrix",
    "Parity",
    "RowPermutation",
    "band_rows",
    "build_kernel_matrix",
    "check_2to4",
    "decode",
    "encode",
    "encode_segment",
    "input_row_permutation",
    "metadata_from_bytes",
    "metadata_to_bytes",
    "sparsity_ratio",
    "sptc_compatible",
    "strided_swap",
    "swap_columns",
    "ExecConfig",
    "DeviceConfig",
    "ExecStats",
    "transform_stencil",
    "execute",
    "naive_apply",
    "verify",
    "report_json",
    "__version__",
]
