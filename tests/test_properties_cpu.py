"""Property tests (hypothesis) of the host-side connectivity: the C++ skeleton
builder against the oracle restatement on random mesh sizes, the invariants of
condense's tables, and the slab partition.  CPU only."""

from __future__ import annotations

import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import mesh_oracle as MO
from paper_2302_10917_b200.mesh import (build_structured_macro_mesh, condense_tables,
                                        elems_per_slab, mesh_tables, slab_partition)

SETTINGS = settings(max_examples=20, deadline=None)


@SETTINGS
@given(d=st.sampled_from([2, 3]), n=st.integers(1, 9))
def test_skeleton_matches_oracle(d, n):
    if d == 3:
        n = min(n, 5)
    o = MO.structured_skeleton(d, n)
    m = build_structured_macro_mesh(d, n, 1)
    for k in ("face_left", "face_right", "elem_face", "face_verts", "elem_verts"):
        assert np.array_equal(getattr(m, k), o[k]), k
    assert np.array_equal(m.face_boundary, o["face_tag"])


@SETTINGS
@given(d=st.sampled_from([2, 3]), n=st.integers(1, 6), neumann_side=st.integers(-1, 3))
def test_condense_table_invariants(d, n, neumann_side):
    if d == 3:
        n = min(n, 4)

    def tagger(x):
        if neumann_side < 0:
            return "D"
        ax, val = divmod(neumann_side, 2)
        return "N" if abs(x[ax % d] - val) < 1e-12 else "D"

    m = build_structured_macro_mesh(d, n, 1, boundary_tagger=tagger)
    tab = mesh_tables(m)
    tab.update(condense_tables(tab))
    uidx, ef, fe, fs = tab["uidx"], tab["elem_ufac"], tab["face_elem"], tab["face_slot"]
    F = tab["F"]
    # unknown faces are the non-Dirichlet ones, numbered in face-id order
    assert F == int((m.face_tag != "D").sum())
    assert np.array_equal(np.sort(uidx[uidx >= 0]), np.arange(F))
    assert np.all(np.diff(np.nonzero(uidx >= 0)[0]) > 0)
    # every side of an unknown face points back at it through its macro's slot
    for u in range(F):
        for c in range(2):
            e, k = fe[u, c], fs[u, c]
            if e < 0:
                assert c == 1
                continue
            assert ef[e, k] == u
    # interior faces have two sides with the lower macro id on the left (mesh.py:235)
    two = fe[:, 1] >= 0
    assert np.all(fe[two, 0] < fe[two, 1])
    # counting KATs: 2-D 3n^2 + 2n faces; 3-D 12n^3 - 6n^2 interior + 12n^2 boundary
    n_faces = m.n_face
    assert n_faces == (3 * n * n + 2 * n if d == 2 else 12 * n ** 3 - 6 * n * n + 12 * n * n)


@SETTINGS
@given(d=st.sampled_from([2, 3]), n=st.integers(1, 40), ranks=st.integers(1, 8))
def test_slab_partition_properties(d, n, ranks):
    N = 2 * n * n if d == 2 else 6 * n ** 3
    per = elems_per_slab(d, n)
    b = slab_partition(N, per, ranks)
    assert b[0] == 0 and b[-1] == N and np.all(np.diff(b) >= 0)
    slabs = N // per
    if slabs % ranks == 0:  # whole slabs, equal shares
        assert np.all(b % per == 0)
        assert len(set(np.diff(b).tolist())) == 1


def test_slab_oracle_equals_whole_mesh_on_complete_faces():
    """oracle.slab_system (the full-size GPU tests' checker): on faces whose sides
    all lie in the slab, the slab's RHS / apply equal the whole mesh's."""
    from oracle import solver_oracle as SO
    from paper_2302_10917_b200 import synthetic as S

    for d, n in ((2, 4), (3, 2)):
        prob = S.make_problem(d, n, 1, 2, seed=3)
        full = SO.system_from_problem(prob).factorize()
        t = prob["t"]
        wf, ff = full.apply(prob["uhat"]), full.rhs()
        N = prob["N"]
        for e0, e1 in ((0, N // 2), (N // 3, N), (N // 4, 3 * N // 4)):
            o, fidx, complete = SO.slab_system(prob, e0, e1)
            o.factorize()
            seg = (fidx[:, None] * t + np.arange(t)).ravel()
            ws = o.apply(prob["uhat"][seg]).reshape(-1, t)
            assert complete.any() and not complete.all()
            assert np.allclose(ws[complete], wf.reshape(-1, t)[fidx[complete]], rtol=0, atol=1e-12)
            assert np.allclose(o.rhs().reshape(-1, t)[complete],
                               ff.reshape(-1, t)[fidx[complete]], rtol=0, atol=1e-12)
            assert not np.allclose(ws[~complete], wf.reshape(-1, t)[fidx[~complete]])


def test_owned_face_generation_matches_whole_mesh_draw():
    """A rank draws only its owned faces' blocks (synthetic_gen.gen_faces_at) --
    the same numbers as the whole-mesh draw, whatever chunks they fall in."""
    from paper_2302_10917_b200 import synthetic_gen as G

    rng = np.random.default_rng(2)
    F = 3 * G.CHUNK + 17
    idx = np.sort(rng.choice(F, 300, replace=False))
    assert np.array_equal(G.gen_faces_at(F, 4, 5, idx), G.gen_faces(F, 4, 5)[idx])
