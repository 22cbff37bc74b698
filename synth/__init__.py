"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NONE of the method's arithmetic (no operator application
inside the ChebyshevT iteration, no truncation): it only builds the inputs the
paper's matrix equation takes (`equation_intro_mat1`) -- the shared CSR
pattern, the six value arrays, the parameter grid / subsets, the
low-rank right-hand side factors -- and the Chebyshev spectrum bounds (the
paper's "Est." harness step). See DESIGN.md "Input recipe".
"""
from .generator import (  # noqa: F401
    CONFIGS,
    Problem,
    config_by_name,
    counter_normal,
    make_problem,
    make_operator,
    parameter_grid,
    split_subsets,
    upper_median_index,
    rhs_factors,
    dense_factor,
)
