"""Seeded synthetic operators of BASELINE.json's configs ("block assembly").

BASELINE.json replaces the reference's FEM assembly (assembly.py:170-322)
with seeded random blocks of the real shapes.  Draw order (fixed here and
recorded in every bench line):

  macros, in chunks of CHUNK ids, rng = numpy PCG64 default_rng([seed, 0, chunk]):
      A_e  = N(0,1)^{Q x Q} + Q*I          (diagonally dominant; ref op.A)
      B_e  = N(0,1)^{nc x Q}               (ref op.C = B_e, op.B = B_e^T)
      R_u  = N(0,1)^{Q}
  unknown faces, in chunks of CHUNK, rng = default_rng([seed, 1, chunk]):
      C_f  = G G^T + 10*I,  G = N(0,1)^{t x t}   (SPD; ref FaceOperator.D)
  uhat = default_rng([seed, 2]).standard_normal(zhat);  R_hat = 0.

Chunking by macro / face id makes every block independent of how the mesh
is partitioned across GPUs.  Q = binom(mp+d, d), t = binom(mp+d-1, d-1),
nc = (d+1) t (fem_basis.py:20-26, costmodel.py:46-58).
"""

from __future__ import annotations

import numpy as np

from .mesh import build_structured_macro_mesh, condense_tables, mesh_tables
from .synthetic_gen import (CHUNK, CONFIGS, block_sizes, gen_faces, gen_faces_at,  # noqa: F401
                            gen_macros, gen_uhat)


def make_problem(d: int, n: int, m: int, p: int, seed: int = 0, with_blocks: bool = True,
                 mesh=None) -> dict:
    """Mesh, condense tables and seeded blocks of one BASELINE config."""
    mesh = mesh or build_structured_macro_mesh(d, n, m)
    Q, t, nc = block_sizes(d, m, p)
    tab = condense_tables(mesh_tables(mesh))
    N, F = mesh.n_elem, tab["F"]
    prob = dict(d=d, n=n, m=m, p=p, seed=seed, Q=Q, t=t, nc=nc, N=N, F=F, zhat=F * t,
                mesh=mesh, elem_face=tab["elem_ufac"], face_elem=tab["face_elem"],
                face_slot=tab["face_slot"], uidx=tab["uidx"])
    if with_blocks:
        A, Be, Ru = gen_macros(N, Q, nc, seed)
        prob.update(A=A, Be=Be, R_u=Ru, D=gen_faces(F, t, seed), R_hat=np.zeros((F, t)),
                    uhat=gen_uhat(F * t, seed))
        # reference views: op.B = B_e^T (Q x nc), op.C = B_e (nc x Q)
        prob["B"] = Be.transpose(0, 2, 1)
        prob["C"] = Be
    return prob


def config_problem(name: str, seed: int = 0, with_blocks: bool = True) -> dict:
    d, n, m, p = CONFIGS[name]
    return make_problem(d, n, m, p, seed=seed, with_blocks=with_blocks)


def algorithmic_bytes_per_apply(N, Q, nc, d, F, t, separate_c=False) -> int:
    """N [8Q^2 + 4Q + 8 nc Q (x2 with separate C) + 16 nc + 4(d+1)]
    + F [8 t^2 + 32 t]."""
    bq = 8 * nc * Q * (2 if separate_c else 1)
    return N * (8 * Q * Q + 4 * Q + bq + 16 * nc + 4 * (d + 1)) + F * (8 * t * t + 32 * t)


def flops_per_apply(N, Q, nc, F, t) -> int:
    return N * (2 * Q * Q + 4 * nc * Q) + F * 2 * t * t


def lu_flops(N, Q) -> float:
    return N * (2.0 / 3.0) * Q**3
