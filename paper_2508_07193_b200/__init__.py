"""B200-native FlashMP hot path (arXiv 2508.07193): drop-in for the reference package
`flashmp`'s preconditioner / solver API, computed by hand-written sm_100a kernels in
libflashmp_b200.so (see include/flashmp_b200.h).

Importing the package needs only numpy/torch; every compute entry point loads the
CUDA library and raises if it (or a GPU) is missing -- there is no CPU fallback.
"""

from .grid import Box, FieldVector, GridMajorVector, dump_field, load_field
from .operators import OperatorParams, apply_curl, apply_double_curl, apply_operator
from .transform import TransformSet, svd_of_difference
from .subdomain import (DegenerateConfigurationError, SubdomainSolverData, analytic_cost, correction_size,
                        cost_report, exact_solve, precompute, solve)
from .schwarz import (BlockLayout, CommunicationError, DistributedOperator, Exchanger, HaloExchanger, Partition,
                      RasPreconditioner, exchange_halo, gather_field, make_partition, make_transport,
                      proc_grid_for, ras_apply, scatter_field, solver_data_for)
from .krylov import SolveReport, SolverConfig, bicgstab, gmres, reduce_dot
from .cn_driver import CnSolver, DeviceCnStepper, EmState, HostStepPipeline, StepFailure, build_rhs, cn_step
from .instrument import BREAKDOWN_CATEGORIES, FlopCounter, NullTimer, PhaseTimer
from ._lib import FlashMPError
from . import reports

__version__ = "0.1.0"
