"""B200-native prior-preconditioned CG sampler (arXiv 1810.12437 hot path).

Drop-in for the reference package `priorcg` on its beta-draw path: the same
public names as pkg/src/priorcg/__init__.py:22-41, backed by hand-written
sm_100a CUDA kernels in libpcgs.so (C ABI: include/pcgs.h).  There is no CPU
fallback: the device entry points raise when the library or the GPU is absent.
"""

__version__ = "0.1.0"

from .sparse import (DenseSymmetric, DimensionCapError, NotPositiveDefiniteError,
                     SparseDesignMatrix, hstack_dense_columns)
from .cg import CGConfig, CGReport, NumericBreakdownError, initial_vector, pcg_solve
from .precond import (DegeneratePreconditionerError, Preconditioner, PreconditionerKind,
                      augmented_prior, gamma_policy, identity_preconditioner,
                      jacobi_preconditioner, prior_preconditioner)
from .sampler import (GaussianTarget, PhiloxGenerator, PrecisionOperator, cg_sample,
                      direct_sample, generate_rhs)
from .polya_gamma import pg_draw, pg_draw_batch, pg_mean
from .gibbs import (BridgeConfig, ChainOutput, GibbsAbortError, HorseshoeConfig, ShrinkageState,
                    gibbs_run)
from .synthdata import SimSpec, simulate_design, simulate_outcomes

__all__ = [
    "BridgeConfig",
    "CGConfig",
    "CGReport",
    "ChainOutput",
    "DenseSymmetric",
    "DegeneratePreconditionerError",
    "DimensionCapError",
    "GaussianTarget",
    "GibbsAbortError",
    "HorseshoeConfig",
    "NotPositiveDefiniteError",
    "NumericBreakdownError",
    "PhiloxGenerator",
    "PrecisionOperator",
    "Preconditioner",
    "PreconditionerKind",
    "ShrinkageState",
    "SimSpec",
    "SparseDesignMatrix",
    "__version__",
    "augmented_prior",
    "cg_sample",
    "direct_sample",
    "gamma_policy",
    "generate_rhs",
    "gibbs_run",
    "hstack_dense_columns",
    "identity_preconditioner",
    "initial_vector",
    "jacobi_preconditioner",
    "pcg_solve",
    "pg_draw",
    "pg_draw_batch",
    "pg_mean",
    "prior_preconditioner",
    "simulate_design",
    "simulate_outcomes",
]
