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

import concurrent.futures as cf
import os
from math import comb

import numpy as np

from .mesh import build_structured_macro_mesh, condense_tables, mesh_tables

CHUNK = 4096

# BASELINE.json configs (d, n, m, p); c5 is the weak-scaling family
CONFIGS = {
    "c1": (2, 8, 2, 2),
    "c2": (2, 128, 4, 3),
    "c3": (3, 16, 2, 3),
    "c4": (3, 24, 3, 3),
    "c5n20": (3, 20, 2, 4),
    "c5n25": (3, 25, 2, 4),
    "c5n32": (3, 32, 2, 4),
    "c5n40": (3, 40, 2, 4),
}


def block_sizes(d: int, m: int, p: int) -> tuple:
    Q = comb(m * p + d, d)
    t = comb(m * p + d - 1, d - 1)
    return Q, t, (d + 1) * t


def _threads(n_chunks: int) -> int:
    return max(1, min(n_chunks, os.cpu_count() or 1, 16))


def gen_macros(N: int, Q: int, nc: int, seed: int = 0, first: int = 0, count: int = None):
    """Blocks of macros [first, first+count): (A, B_e, R_u)."""
    count = N - first if count is None else count
    A = np.empty((count, Q, Q))
    Be = np.empty((count, nc, Q))
    Ru = np.empty((count, Q))
    c0, c1 = first // CHUNK, (first + count + CHUNK - 1) // CHUNK

    def work(c):
        lo, hi = c * CHUNK, min((c + 1) * CHUNK, N)
        rng = np.random.default_rng([seed, 0, c])
        a = rng.standard_normal((hi - lo, Q, Q))
        a[:, np.arange(Q), np.arange(Q)] += Q
        b = rng.standard_normal((hi - lo, nc, Q))
        r = rng.standard_normal((hi - lo, Q))
        s0, s1 = max(lo, first), min(hi, first + count)
        if s1 > s0:
            A[s0 - first:s1 - first] = a[s0 - lo:s1 - lo]
            Be[s0 - first:s1 - first] = b[s0 - lo:s1 - lo]
            Ru[s0 - first:s1 - first] = r[s0 - lo:s1 - lo]

    with cf.ThreadPoolExecutor(_threads(c1 - c0)) as ex:
        list(ex.map(work, range(c0, c1)))
    return A, Be, Ru


def gen_faces(F: int, t: int, seed: int = 0, first: int = 0, count: int = None):
    count = F - first if count is None else count
    D = np.empty((count, t, t))
    c0, c1 = first // CHUNK, (first + count + CHUNK - 1) // CHUNK

    def work(c):
        lo, hi = c * CHUNK, min((c + 1) * CHUNK, F)
        rng = np.random.default_rng([seed, 1, c])
        G = rng.standard_normal((hi - lo, t, t))
        Dc = np.matmul(G, G.transpose(0, 2, 1))
        Dc[:, np.arange(t), np.arange(t)] += 10.0
        s0, s1 = max(lo, first), min(hi, first + count)
        if s1 > s0:
            D[s0 - first:s1 - first] = Dc[s0 - lo:s1 - lo]

    with cf.ThreadPoolExecutor(_threads(c1 - c0)) as ex:
        list(ex.map(work, range(c0, c1)))
    return D


def gen_uhat(zhat: int, seed: int = 0) -> np.ndarray:
    return np.random.default_rng([seed, 2]).standard_normal(zhat)


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
