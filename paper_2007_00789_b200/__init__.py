"""B200-native spaND: sparsified nested-dissection factorization + PCG.

Drop-in for the factorize / preconditioner-apply / PCG path of the
reference package ``spdkit`` (`/root/reference/pkg/src/spdkit/__init__.py`):
same names, argument meaning and error types; the numerical work runs in the
sm_100a extension ``libspand_b200.so`` (C-ABI in ``include/spand_b200.h``).
"""

from .dense import (
    RRQRResult,
    SchemeKind,
    cholesky,
    rrqr_sparsify,
    tri_inverse,
    tri_solve,
)
from .errors import (
    AsymmetricValues,
    Breakdown,
    DimensionMismatch,
    InputError,
    NativeUnavailable,
    NonFinite,
    NonpositiveDiagonal,
    NotSPD,
    NotSymmetricReal,
    NumericalError,
    PanelTooLarge,
    ParseError,
    RhoNotOne,
    SingularTriangular,
    SpdkitError,
)
from .factorize import (
    Factorization,
    apply_inv,
    apply_inv_t,
    factorize,
    load_factor,
    memory_ratio,
    save_factor,
)
from .krylov import SolveReport, cg_bound_rate, default_maxit, pcg, pcg_multi
from .partition import Cluster, PartitionHierarchy, build_hierarchy, default_levels
from .schemes import (
    OpKind,
    SparsificationResult,
    local_error,
    make_elimination,
    make_scaling,
    make_sparsification,
)
from .sparse import (
    SparseSymMatrix,
    baseline_problem,
    c5_problem,
    diffusion_fv,
    diffusion_fv_device,
    elasticity_q1,
    from_coo,
    jacobi_prescale,
    laplacian_2d,
    laplacian_3d,
    log_uniform_block_field,
    read_matrix_market,
    rigid_body_modes,
    write_matrix_market,
)

__version__ = "0.1.0"
