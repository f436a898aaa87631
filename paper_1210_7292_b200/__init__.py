"""paper_1210_7292_b200 — B200-native M2L application for the Chebyshev
black-box FMM (arXiv 1210.7292), a drop-in for the reference package's
``M2LHandler`` precompute/apply API (chebfmm/m2l.py).

Product path: host precompute (numerics.py) -> device operator cache ->
CUDA tile kernels for sm_100a behind the C ABI in include/chebm2l.h
(libchebm2l.so, loaded by _native.py).  No CPU fallback.
"""

from .m2l import (
    DEFAULT_BUDGET_BYTES,
    VARIANTS,
    B200M2LHandler,
    BudgetExceededError,
    M2LHandler,
    PrecomputeIncompleteError,
    make_handler,
)
from .numerics import (
    AffineMap,
    ChebyshevGrid,
    Kernel,
    LowRankFactors,
    aca,
    aca_plus_svd,
    assemble_for_transfer,
    cheb_roots,
    helmholtz_kernel,
    laplace_kernel,
    truncated_svd,
)
from .symmetry import (
    PermutationSpec,
    SymmetryMap,
    canonicalize,
    full_far_field_vectors,
    inverse_permutation_table,
    permutation_table,
)

__all__ = [
    "DEFAULT_BUDGET_BYTES",
    "VARIANTS",
    "B200M2LHandler",
    "BudgetExceededError",
    "M2LHandler",
    "PrecomputeIncompleteError",
    "make_handler",
    "AffineMap",
    "ChebyshevGrid",
    "Kernel",
    "LowRankFactors",
    "aca",
    "aca_plus_svd",
    "assemble_for_transfer",
    "cheb_roots",
    "helmholtz_kernel",
    "laplace_kernel",
    "truncated_svd",
    "PermutationSpec",
    "SymmetryMap",
    "canonicalize",
    "full_far_field_vectors",
    "inverse_permutation_table",
    "permutation_table",
]
