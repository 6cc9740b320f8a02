"""The C-ABI library on a CPU-only host: it loads, exports every symbol the
header declares, and its host-side connectivity builder is bit-exact with the
reference skeleton.  No GPU compute is called here."""

from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, golden
from oracle import mesh_oracle as MO
from paper_2302_10917_b200 import _lib
from paper_2302_10917_b200.mesh import (build_structured_macro_mesh, condense_tables,
                                        mesh_tables, slab_partition)

HEADER = ROOT / "include" / "mehdg_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(mh_[a-z0-9_]+)\s*\(", text)) - {"mh_op_fn"})


def test_header_symbols_exported():
    syms = declared_symbols()
    assert len(syms) > 20
    lib = C.CDLL(str(_lib.LIB_PATH))
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(_lib.SIGNATURES) == syms


def test_library_is_sm100a():
    data = _lib.LIB_PATH.read_bytes()
    assert b"sm_100a" in data


def test_device_count_does_not_fail():
    assert _lib.device_count() >= 0


@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
def test_cpp_skeleton_2d_bit_exact_with_reference(n):
    g = golden("skeleton_2d.npz")
    m = build_structured_macro_mesh(2, n, 2)
    assert np.array_equal(m.face_left, g[f"n{n}_face_left"])
    assert np.array_equal(m.face_right, g[f"n{n}_face_right"])
    assert np.array_equal(m.face_boundary, g[f"n{n}_face_tag"])
    assert np.array_equal(m.elem_verts, g[f"n{n}_elem_verts"])
    assert np.array_equal(m.elem_face, g[f"n{n}_elem_face"])
    assert np.array_equal(m.vertices_lattice, g[f"n{n}_verts"])


@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_cpp_kuhn_tets_bit_exact_with_reference(n):
    g = golden("kuhn_3d.npz")
    m = build_structured_macro_mesh(3, n, 2)
    assert np.array_equal(m.elem_verts, g[f"n{n}_elem_verts"])
    assert np.array_equal(m.vertices_lattice, g[f"n{n}_verts"])


@pytest.mark.parametrize("d,n", [(2, 16), (2, 33), (3, 2), (3, 5), (3, 8)])
def test_cpp_skeleton_matches_oracle(d, n):
    o = MO.structured_skeleton(d, n)
    m = build_structured_macro_mesh(d, n, 2)
    for k in ("face_left", "face_right", "elem_face", "face_verts", "elem_verts"):
        assert np.array_equal(getattr(m, k), o[k]), k
    assert np.array_equal(m.face_boundary, o["face_tag"])


def test_cpp_condense_tables_match_reference_c1():
    g = golden("synthetic_c1.npz")
    m = build_structured_macro_mesh(2, 8, 2)
    tab = condense_tables(mesh_tables(m))
    fid = np.nonzero(tab["uidx"] >= 0)[0]
    assert np.array_equal(fid, g["offsets_fid"])
    t = 5
    gi = []
    for e in range(m.n_elem):
        for u in tab["elem_ufac"][e]:
            if u >= 0:
                gi.extend(range(u * t, (u + 1) * t))
    assert np.array_equal(np.array(gi), g["gather_idx_concat"])


def test_reference_mesh_duck_typing():
    """mesh_tables accepts any MacroMesh-like object (skeleton/sides())."""
    m = build_structured_macro_mesh(2, 4, 1)
    sk_tables = mesh_tables(m)

    class Duck:
        skeleton = m.skeleton
        macro_elements = m.macro_elements
        d = 2

    duck = mesh_tables(Duck())
    for k in ("face_unknown", "elem_face", "face_left", "face_right"):
        assert np.array_equal(np.asarray(sk_tables[k]), np.asarray(duck[k])), k


def test_boundary_tagger_neumann_faces_become_unknowns():
    m = build_structured_macro_mesh(2, 3, 1, boundary_tagger=lambda x: "N" if x[0] < 1e-12 else "D")
    tab = condense_tables(mesh_tables(m))
    assert tab["F"] == 3 * 9 - 2 * 3 + 3
    one_sided = (tab["face_elem"][:, 1] < 0).sum()
    assert one_sided == 3


def test_bad_arguments_raise_value_error():
    with pytest.raises(ValueError):
        build_structured_macro_mesh(4, 2, 1)
    with pytest.raises(ValueError):
        build_structured_macro_mesh(2, 0, 1)


def test_slab_partition():
    b = slab_partition(2 * 16 * 16, 32, 4)
    assert list(b) == [0, 128, 256, 384, 512]
    b = slab_partition(6 * 25**3, 6 * 25 * 25, 2)  # 25 x-slabs on 2 ranks: whole slabs 12/13
    assert b[1] % (6 * 25 * 25) == 0 and b[2] == 6 * 25**3
    b = slab_partition(10, 0, 3)
    assert list(b) == [0, 3, 6, 10]


def test_create_without_gpu_fails_loudly():
    if _lib.device_count() > 0:
        pytest.skip("GPU present")
    h = C.c_void_p()
    st = _lib.lib.mh_create(0, 3, 2, 15, 5, 1, C.byref(h))
    assert st == _lib.MH_E_CUDA


@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
def test_export_text_matches_reference(n):
    """mesh.py:479-490 dump of our C++-built mesh equals the reference's, byte for byte."""
    import paper_2302_10917_b200 as P

    g = golden("skeleton_2d.npz")
    ref = bytes(g[f"n{n}_export_text"]).decode()
    assert P.export_text(build_structured_macro_mesh(2, n, 2)) == ref


def test_report_csv_round_trip(tmp_path):
    """17-significant-digit CSV (bench.py:328-379) round-trips report records."""
    import paper_2302_10917_b200 as P

    rows = [{"p": 3, "m": 4, "n": 128, "tol": 1e-10, "converged": True,
             "t_init_s": 0.1 + 0.2, "lbf": 1.0, "mode": "mf"}]
    cols = list(rows[0])
    path = tmp_path / "r.csv"
    P.write_csv(rows, cols, str(path))
    back = P.read_csv(str(path))
    assert back == rows
    assert P.rows_to_csv(rows, cols).splitlines()[1].split(",")[5] == "0.30000000000000004"


def test_solver_config_validation():
    import paper_2302_10917_b200 as P

    for bad in (dict(tol=0.0), dict(tol=1.0), dict(preconditioner="ilu"), dict(mode="x")):
        with pytest.raises(ValueError):
            P.SolverConfig(**bad)
    cfg = P.SolverConfig()
    assert (cfg.tol, cfg.restart, cfg.maxiter, cfg.preconditioner, cfg.mode) == \
        (1e-6, 100, 10000, "dinv", "mf")


def test_worker_pool_static_partition():
    """schur_solver.py:59-102: round-robin items, results independent of workers."""
    import paper_2302_10917_b200 as P

    items = list(range(37))
    ref = [x * x + 1 for x in items]
    for w in (1, 2, 8):
        pool = P.WorkerPool(w)
        seen = []
        assert pool.map(lambda x: (seen.append(x), x * x + 1)[1], items) == ref
        assert sorted(seen) == items and pool.busy.shape == (w,)
        assert 0.0 < pool.lbf <= 1.0
        pool.close()


def test_singular_exceptions_carry_ids():
    import paper_2302_10917_b200 as P

    assert P.SingularLocalBlock(7).args[0] == 7
    assert P.SingularFaceBlock(3).args[0] == 3
