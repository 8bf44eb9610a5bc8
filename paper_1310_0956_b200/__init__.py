"""B200-native hot path of the WMG-preconditioned Krylov tomography solver
(arXiv 1310.0956), a drop-in for the reference package ``wmgtomo``'s public
solver/operator API (/root/reference/pkg/src/wmgtomo/__init__.py:6-18).

Compute runs in hand-written sm_100a kernels (``lib/libwmgb200.so``, C ABI in
``include/wmgb200.h``); PyTorch only provides HBM buffers, streams and
``torch.distributed``.  There is no CPU fallback.
"""

__version__ = "0.1.0"

from .geometry import (Geometry, LineProjector, apply, apply_transpose,  # noqa: F401
                       build_geometry, build_projector)
from .multilevel import (BAND_IDS, IntergridSet, WmgHierarchy, WmgNode,  # noqa: F401
                         build_intergrid_set, build_wmg_hierarchy,
                         classical_tg_preconditioner, haar_scaling_1d,
                         haar_wavelet_1d, wmg_preconditioner, wtg_apply)
from .phantom import (add_gaussian_noise, add_noise, error_metrics,  # noqa: F401
                      poisson_log_data, random_ellipses, seeded_uniform, shepp_logan)
from .solvers import (BREAKDOWN_REL_TOL, STATUS_BREAKDOWN, STATUS_CONVERGED,  # noqa: F401
                      STATUS_MAX_ITERATIONS, ConvergenceRecord, SirtScaling, SolverConfig,
                      bicgstab_solve, cgls_solve, find_kopt, gmres_solve, normal_operator,
                      sirt_scaling, sirt_solve)
from .sparse_kernels import (DenseFactorization, DimensionMismatchError,  # noqa: F401
                             NotPositiveDefiniteError, cholesky_factor, cholesky_solve)
