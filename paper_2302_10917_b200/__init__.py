"""B200-native macro-element Schur-complement operator (arXiv 2302.10917).

Drop-in for the hot path of the reference package ``mehdg``
(``mehdg.schur_solver``): the same names and signatures, with the numerics
in hand-written sm_100a CUDA kernels (libmehdg_b200.so) behind a C-ABI.
"""

from .assembly import FaceOperator, LocalOperators, operators_from_problem
from .mesh import (
    FaceSide,
    MacroElement,
    SkeletonFace,
    StructuredMacroMesh,
    build_structured_macro_mesh,
    condense_tables,
    mesh_tables,
)
from .schur_solver import (
    CondensedSystem,
    Preconditioner,
    SchurOperator,
    SingularFaceBlock,
    SingularLocalBlock,
    Solution,
    SolveReport,
    SolverConfig,
    WorkerPool,
    apply_preconditioner,
    apply_schur,
    apply_schur_mb,
    assemble_schur_explicit,
    condense,
    condense_arrays,
    form_element_schur,
    gmres,
    local_factors,
    reconstruct_interior,
    solve,
    solve_condensed,
)

__version__ = "0.1.0"
