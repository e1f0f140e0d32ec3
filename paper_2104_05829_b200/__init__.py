"""paper_2104_05829_b200 -- B200-native hot path of NekRS (arXiv 2104.05829):
the matrix-free spectral-element operator w_L = QQ^T Z_L u_L inside the
pressure PCG (BK5 stiffness apply, gslib-style gather-scatter, fused CG).

Public API mirrors the reference's ``nekmini`` operator contracts
(/root/reference/SPEC.md): basis, mesh, gather_scatter, kernels, solvers,
partition.  Compute runs in libnekb200.so (hand-written sm_100a CUDA, C ABI in
include/nekb200.h); PyTorch only owns device buffers and streams.
"""

from . import (basis, distributed, gather_scatter, kernels, mesh, multigrid,  # noqa: F401
               partition, projection, schwarz, solvers)
from ._lib import (ContractError, NativeLibraryError, UnsupportedOrderError,  # noqa: F401
                   LIB_PATH)
from .basis import InvalidOrderError, SpectralBasis, gll_rule, interp_matrix  # noqa: F401
from .gather_scatter import gs_op, gs_op_overlapped, gs_setup  # noqa: F401
from .kernels import (apply_helmholtz_local, apply_mass, apply_stiffness_local,  # noqa: F401
                      extract_diagonal, inner_product, select_kernel_variant)
from .mesh import (Mesh, assign_global_ids, build_box_mesh, geometric_factors,  # noqa: F401
                   read_hexmesh, write_hexmesh)
from .multigrid import (MultigridHierarchy, MultigridPCG, chebyshev_smooth,  # noqa: F401
                        coarse_solve, pmg_preconditioner)
from .partition import rcb  # noqa: F401
from .projection import ProjectedSolver, ProjectionSpace, project_guess  # noqa: F401
from .schwarz import SchwarzSmoother, fdm_local_solve, schwarz_smooth  # noqa: F401
from .solvers import (BreakdownError, FusedPCG, FusedPCG3, HelmholtzVectorSolver,  # noqa: F401
                      JacobiPreconditioner, PoissonOperator, pcg)

__version__ = "1.0.0"
