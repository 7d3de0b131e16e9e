"""B200-native generalized-LDL^T inertia engine for rank-structured matrices.

Drop-in for the hot path of the reference package `h2slice`
(arXiv 2311.08618): the inertia of A - mu I for an H2 / HSS / BLR2 matrix A,
and the k-th eigenvalue by bisection on that inertia.  Public names follow
the reference (`h2slice/__init__.py`); the factorization runs in
libh2ldl.so (hand-written sm_100a CUDA behind the C ABI in include/h2ldl.h).
"""

from .bisection import (
    EPS_EV_DEFAULT,
    EigenvalueEstimate,
    InertiaCache,
    default_interval,
    multisection,
    slice_range,
    slice_spectrum,
)
from .cluster import (
    WEAK,
    Admissibility,
    BlockStructure,
    ClusterTree,
    build_tree,
    classify,
    construction_partners,
    flat_structure,
    strong,
)
from .errors import (
    Breakdown,
    ConfigError,
    H2SliceError,
    IncompleteSpectrum,
    InertiaUnstable,
    NativeError,
    NotInInterval,
    OracleTooLarge,
    ShiftHitEigenvalue,
)
from .geometry import (
    DenseKernel,
    HoppingKernel,
    InverseDistanceKernel,
    KernelFn,
    LaplaceKernel,
    LogKernel,
    PointCloud,
    YukawaKernel,
    generate_circle,
    generate_grid,
    laplace_kernel,
    load_point_cloud,
    matrix_kernel,
    save_point_cloud,
    sfc_order,
)
from .h2matrix import (
    BasisSplit,
    RankStructuredMatrix,
    construct,
    gershgorin_interval,
    load_payload,
    reconstruct_dense,
    rrqr_truncated,
    save_payload,
    shift_diagonal,
)
from .ldl import GldlFactorization, InertiaCount, generalized_ldl, inertia, inertia_batch

__version__ = "0.1.0"
BACKEND = "cuda-sm100a"
