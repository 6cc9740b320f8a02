"""B200-native macro-element Schur-complement operator (arXiv 2302.10917).

Drop-in for the hot path of the reference package ``mehdg``
(``mehdg.schur_solver``): the same names and signatures, with the numerics
in hand-written sm_100a CUDA kernels (libmehdg_b200.so) behind a C-ABI.

Names are resolved lazily so that ``paper_2302_10917_b200._build`` can
(re)build the library without loading a stale copy of it.
"""

from importlib import import_module

__version__ = "0.1.0"

_EXPORTS = {
    "assembly": ["DeviceBlocks", "FaceOperator", "LocalOperators", "ProblemData",
                 "StabilizationConfig", "assemble_system_device", "manufactured_tanh",
                 "operators_from_problem"],
    "io": ["export_text", "read_csv", "rows_to_csv", "write_csv"],
    "mesh": ["FaceSide", "MacroElement", "SkeletonFace", "StructuredMacroMesh",
             "build_structured_macro_mesh", "condense_tables", "mesh_tables"],
    "schur_solver": ["CondensedSystem", "Preconditioner", "SchurOperator", "SingularFaceBlock",
                     "SingularLocalBlock", "Solution", "SolveReport", "SolverConfig",
                     "WorkerPool", "apply_preconditioner", "apply_schur", "apply_schur_many", "apply_schur_mb",
                     "assemble_schur_explicit", "condense", "condense_arrays",
                     "form_element_schur", "gmres", "local_factors", "reconstruct_interior",
                     "solve", "solve_condensed"],
}
_WHERE = {name: mod for mod, names in _EXPORTS.items() for name in names}
__all__ = sorted(_WHERE)


def __getattr__(name):
    mod = _WHERE.get(name)
    if mod is None:
        raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
    value = getattr(import_module(f".{mod}", __name__), name)
    globals()[name] = value
    return value


def __dir__():
    return sorted(list(globals()) + __all__)
