"""B200-native (sm_100a) hot path of the ADMoM non-negative CP solver.

Drop-in for the reference package's NTF entry point (``cpadmm.fit``,
reference solver.py:340) and its multi-device analogue
(``cpadmm.distributed_fit``, mesh.py:331): same argument and return types,
results matching the reference CPU implementation on the same seeded inputs.
The per-mode update — dense MTTKRP, Gram-Hadamard + ridge Cholesky, and the
fused row solve / projection / dual step — runs in hand-written CUDA kernels
behind the C ABI declared in ``include/ntf_b200.h``.
"""

from .constraints import ConstraintSpec
from .distributed import PartitionPlan, ShardedTensor, distributed_fit
from .solver import (
    FitResult,
    InvalidPenaltyError,
    Residuals,
    SolverConfig,
    SolverState,
    derive_seed,
    fit,
    init_state,
    iterate,
    mttkrp_factors,
    release_plan_cache,
)
from . import tensor_io  # noqa: F401
from .tensors import CooTensor, DenseTensor, KruskalModel

__version__ = "0.1.0"

__all__ = [
    "ConstraintSpec",
    "CooTensor",
    "DenseTensor",
    "FitResult",
    "InvalidPenaltyError",
    "KruskalModel",
    "PartitionPlan",
    "Residuals",
    "SolverConfig",
    "SolverState",
    "derive_seed",
    "distributed_fit",
    "ShardedTensor",
    "fit",
    "init_state",
    "release_plan_cache",
    "iterate",
    "mttkrp_factors",
]
