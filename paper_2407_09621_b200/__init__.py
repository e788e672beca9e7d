"""B200-native (sm_100a) SIPG sum-factorisation hot path of arXiv 2407.09621.

Drop-in for the reference package ``sumfact``'s operator/solver API
(apply_operator, MultigridPreconditioner, restrict/prolongate, fgmres/gmres,
run_solve).  All compute runs in libsumfact_b200.so; there is no CPU fallback.
"""
__version__ = "0.1.0"

from .precision import (PrecisionMode, relative_error, HalfRangeError, EcPair, to_half, from_half,  # noqa: F401
                        demote16, ec_split, ec_matmul)
from .core import contract_batch, contract_mode  # noqa: F401
from .discretization import (MeshHierarchy, build_hierarchy, apply_operator, materialize_operator,  # noqa: F401
                             assemble_rhs, interpolate, l2_error, h1_seminorm_error, sine_product_problem,
                             save_vector, load_vector)
from .multigrid import (MultigridPreconditioner, VCycleConfig, PatchSolver, default_ordering,  # noqa: F401
                        restrict, prolongate, patch_inverse_apply)
from .krylov import fgmres, gmres, SolveReport  # noqa: F401
from .experiments import run_solve, convergence_study, error_profile  # noqa: F401
