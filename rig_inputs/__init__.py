"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no scaling, no products, no
cutsize).  It only draws sparse matrices and partitions with the shapes of the
paper's workloads (BASELINE.json ``configs``), so both
sides of every parity test read identical arrays.
"""
from .configs import (  # noqa: F401
    Workload,
    CONFIG_NAMES,
    make,
    make_small,
    stencil2d,
    stencil3d,
    powerlaw,
    banded,
    dense_columns,
    uniform_rows,
    part_contiguous,
    part_random_balanced,
    part_random_iid,
    from_dense,
    from_triplets,
)
