"""B200-native batched Boys-function evaluator (Laikov, arXiv 2504.07637).

F_n(x) = c_n / (x + Q~_n(x)^{n+1/2} e^{-x})^{n+1/2} with a root-factored
rational Q~_n, the asymptote c_n x^{-(n+1/2)} past the cut-off z_nb, and the
downward recursion for F_0..F_{n-1}; evaluated by hand-written sm_100a CUDA
kernels behind the C ABI in include/boys.h.

Public API (mirrors the reference's SPEC'd ``kernel`` module):
    boys, boys_ragged, ragged_offsets, eval_batch, eval_fn, eval_with_split,
    EvalRequest, EvalResult, max_order; and the fused consumer hermite_coulomb
"""

from .kernel import (  # noqa: F401
    EvalRequest,
    EvalResult,
    boys,
    boys_ragged,
    eval_batch,
    eval_fn,
    eval_with_split,
    hermite_coulomb,
    max_order,
    ragged_offsets,
)

__version__ = "0.2.0"   # matches libboys (BOYS_VERSION)
