"""Slab partition and halo plans for multi-GPU runs.

Rank r owns the contiguous macro range [elem_begin[r], elem_begin[r+1])
(whole mesh rows in 2-D -- 2n macros per row, mesh.py:376-387 -- and whole
x-slabs in 3-D -- 6n^2 tets, mesh.py:407-417 -- when they divide evenly)
and every unknown face whose LEFT (lower-id, mesh.py:235) macro it owns.
Because macro ids increase across slabs, the right side of an owned face is
on the same or a higher rank, so the halo of rank r is exactly the faces
whose right macro is on r and whose left macro is on a lower rank.

The plan reproduces the reference's left-then-right face reduction
(schur_solver.py:234-241, 284-290): the owner subtracts its own left
contribution first and the neighbour's right contribution second, so a
multi-GPU apply is bitwise identical to the single-GPU one.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .mesh import elems_per_slab, slab_partition


@dataclass
class RankPlan:
    rank: int
    nranks: int
    e0: int
    e1: int
    owned: np.ndarray          # global unknown-face ids owned here (ascending)
    halo: np.ndarray           # global ids of halo faces, grouped by owner then id
    elem_ufac: np.ndarray      # (N_loc, nfe) local trace index or -1
    face_elem: np.ndarray      # (F_own, 2) local macro / N_loc + extra slot / -1
    face_slot: np.ndarray      # (F_own, 2)
    send_face: np.ndarray      # local owned indices, grouped by destination rank
    send_count: np.ndarray     # (nranks,)
    recv_count: np.ndarray     # (nranks,) halo faces received from each owner
    vret_slot: np.ndarray      # local v-slot (e*nfe + k) per halo face, grouped by owner
    vret_count: np.ndarray     # (nranks,)
    vrecv_count: np.ndarray    # (nranks,) v segments received from each neighbour
    vrecv_face: np.ndarray     # global ids of the faces whose right v arrives here

    @property
    def n_local(self) -> int:
        return self.e1 - self.e0

    @property
    def F_own(self) -> int:
        return int(self.owned.size)

    @property
    def F_halo(self) -> int:
        return int(self.halo.size)


def partition(d: int, n: int, n_elem: int, nranks: int) -> np.ndarray:
    return slab_partition(n_elem, elems_per_slab(d, n), nranks)


def rank_plan(elem_ufac: np.ndarray, face_elem: np.ndarray, face_slot: np.ndarray,
              elem_begin: np.ndarray, rank: int) -> RankPlan:
    """Plan of one rank from the GLOBAL condense tables."""
    elem_begin = np.asarray(elem_begin, np.int64)
    nranks = elem_begin.size - 1
    nfe = elem_ufac.shape[1]
    F = face_elem.shape[0]

    def rank_of(e):
        return np.searchsorted(elem_begin, e, side="right") - 1

    L, Rm = face_elem[:, 0].astype(np.int64), face_elem[:, 1].astype(np.int64)
    owner = rank_of(L)
    rr = np.where(Rm >= 0, rank_of(np.maximum(Rm, 0)), -1)
    if np.any((Rm >= 0) & (rr < owner)):
        raise ValueError("a face's right macro lies on a lower rank than its left macro")
    e0, e1 = int(elem_begin[rank]), int(elem_begin[rank + 1])
    owned = np.nonzero(owner == rank)[0]
    halo = np.nonzero((rr == rank) & (owner != rank))[0]
    halo = halo[np.lexsort((halo, owner[halo]))]
    loc = np.full(F, -1, np.int64)
    loc[owned] = np.arange(owned.size)
    loc[halo] = owned.size + np.arange(halo.size)
    eu = elem_ufac[e0:e1].astype(np.int64)
    elem_ufac_loc = np.where(eu >= 0, loc[np.maximum(eu, 0)], -1)
    if np.any((eu >= 0) & (elem_ufac_loc < 0)):
        raise ValueError("macro references a face that is neither owned nor halo")
    n_loc = e1 - e0

    # v-slot contributions arriving from higher ranks (right side remote)
    remote_right = owned[(rr[owned] >= 0) & (rr[owned] != rank)]
    vrecv = remote_right[np.lexsort((remote_right, rr[remote_right]))]
    extra = np.full(F, -1, np.int64)
    extra[vrecv] = np.arange(vrecv.size)

    fe = np.full((owned.size, 2), -1, np.int64)
    fs = np.full((owned.size, 2), -1, np.int64)
    fe[:, 0] = L[owned] - e0
    fs[:, 0] = face_slot[owned, 0]
    same = rr[owned] == rank
    fe[same, 1] = Rm[owned][same] - e0
    fs[same, 1] = face_slot[owned, 1][same]
    rem = (rr[owned] >= 0) & ~same
    fe[rem, 1] = n_loc + extra[owned[rem]]
    fs[rem, 1] = 0

    send_face, send_count = [], np.zeros(nranks, np.int32)
    for q in range(nranks):
        if q == rank:
            continue
        s = owned[rr[owned] == q]
        send_face.append(loc[s])
        send_count[q] = s.size
    recv_count = np.bincount(owner[halo], minlength=nranks).astype(np.int32)
    vret_slot = (Rm[halo] - e0) * nfe + face_slot[halo, 1]
    vret_count = recv_count.copy()
    vrecv_count = np.bincount(rr[vrecv], minlength=nranks).astype(np.int32) if vrecv.size \
        else np.zeros(nranks, np.int32)
    return RankPlan(
        rank=rank, nranks=nranks, e0=e0, e1=e1, owned=owned, halo=halo,
        elem_ufac=elem_ufac_loc.astype(np.int32), face_elem=fe.astype(np.int32),
        face_slot=fs.astype(np.int32),
        send_face=(np.concatenate(send_face) if send_face else np.zeros(0, np.int64)).astype(np.int32),
        send_count=send_count, recv_count=recv_count,
        vret_slot=vret_slot.astype(np.int32), vret_count=vret_count.astype(np.int32),
        vrecv_count=vrecv_count, vrecv_face=vrecv)
