"""Seeded synthetic blocks of BASELINE.json's configs -- pure numpy.

The draw order is documented in ``synthetic.py``.  This module imports
nothing from the package (no ctypes, no CUDA library), so that bench.py's
``--impl reference`` arm can feed the unmodified reference solver exactly the
same blocks as the GPU path without loading ``libmehdg_b200.so`` (it loads
this file by path).
"""

from __future__ import annotations

import concurrent.futures as cf
import os
from math import comb

import numpy as np

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
        s0, s1 = max(lo, first), min(hi, first + count)
        if s0 == lo and s1 == hi:
            # whole chunk in range: draw straight into the outputs (the same
            # C-order stream as the temporary-array form below, no copies)
            a = A[s0 - first:s1 - first]
            rng.standard_normal(out=a)
            a[:, np.arange(Q), np.arange(Q)] += Q
            rng.standard_normal(out=Be[s0 - first:s1 - first])
            rng.standard_normal(out=Ru[s0 - first:s1 - first])
            return
        a = rng.standard_normal((hi - lo, Q, Q))
        a[:, np.arange(Q), np.arange(Q)] += Q
        b = rng.standard_normal((hi - lo, nc, Q))
        r = rng.standard_normal((hi - lo, Q))
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


def gen_faces_at(F: int, t: int, seed: int, idx) -> np.ndarray:
    """The face blocks of the unknown faces `idx` only (a rank's owned faces):
    each CHUNK of faces that holds one of them is drawn once, the same stream
    as gen_faces(F, t, seed)[idx]."""
    idx = np.asarray(idx, dtype=np.int64)
    out = np.empty((idx.size, t, t))
    which = idx // CHUNK
    chunks = np.unique(which)

    def work(c):
        lo = int(c) * CHUNK
        Dc = gen_faces(F, t, seed, lo, min(CHUNK, F - lo))
        sel = which == c
        out[sel] = Dc[idx[sel] - lo]

    with cf.ThreadPoolExecutor(_threads(chunks.size)) as ex:
        list(ex.map(work, chunks))
    return out
