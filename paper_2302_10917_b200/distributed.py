"""Multi-GPU driver: one rank per GPU, slab-partitioned macros, NCCL halos.

`RankSystem` is the per-rank counterpart of ``CondensedSystem``: it uploads
the rank's macros, owned faces and halo plan (partition.rank_plan) to
libmehdg_b200, which then runs the apply / RHS / GMRES with the uhat-halo,
v-return and dot-product exchanges over NCCL (mh_comm_init).  torch.distributed
only carries the 128-byte NCCL unique id at start-up.

`group_apply` runs all ranks of a partition inside one process on one GPU
(device copies instead of NCCL) so that the halo plans and kernels can be
checked bitwise against the single-GPU apply without a multi-GPU box.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import check, lib, ptr
from .partition import RankPlan
from .schur_solver import MH_E_SINGULAR_FACE, MH_E_SINGULAR_LOCAL, SingularFaceBlock, \
    SingularLocalBlock, _Handle, _torch


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib.mh_comm_unique_id(buf), "mh_comm_unique_id")
    return buf.raw


def broadcast_unique_id(rank: int, device: int) -> bytes:
    """Rank 0 creates the NCCL id; torch.distributed broadcasts it."""
    torch = _torch()
    import torch.distributed as dist

    t = torch.zeros(128, dtype=torch.uint8, device=f"cuda:{device}"
                    if dist.get_backend() == "nccl" else "cpu")
    if rank == 0:
        t.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(t, src=0)
    return bytes(t.cpu().numpy().tobytes())


class RankSystem:
    """The slab of one rank on one device."""

    def __init__(self, prob: dict, plan: RankPlan, device: int = 0, comm_id: bytes = None,
                 blocks: dict = None):
        torch = _torch()
        self.plan, self.device = plan, device
        self.t, self.Q, self.nfe = prob["t"], prob["Q"], prob["d"] + 1
        self.N, self.F = plan.n_local, plan.F_own
        self.zhat = self.F * self.t
        self._h = _Handle(device, self.nfe, self.N, self.Q, self.t, self.F)
        h = self._h.h
        check(lib.mh_set_halo(h, plan.nranks, plan.rank, ptr(_i32(plan.send_face)),
                              ptr(_i32(plan.send_count)), ptr(_i32(plan.recv_count)),
                              ptr(_i32(plan.vret_slot)), ptr(_i32(plan.vret_count)),
                              ptr(_i32(plan.vrecv_count))), "mh_set_halo")
        # a communicator is used whenever one is given (with one rank too: the
        # NCCL calls then run on a single-GPU box, tests/test_gpu_multislab.py)
        self.has_comm = comm_id is not None
        if self.has_comm:
            idb = C.create_string_buffer(comm_id, 128)
            check(lib.mh_comm_init(h, idb, plan.nranks, plan.rank), "mh_comm_init")
        check(lib.mh_upload_connectivity(h, ptr(_i32(plan.elem_ufac)), ptr(_i32(plan.face_elem)),
                                         ptr(_i32(plan.face_slot))), "mh_upload_connectivity")
        if blocks is None:
            e0, e1 = plan.e0, plan.e1
            blocks = dict(A=prob["A"][e0:e1], Be=prob["Be"][e0:e1], R_u=prob["R_u"][e0:e1],
                          D=prob["D"][plan.owned], R_hat=prob["R_hat"][plan.owned])
        A = np.ascontiguousarray(blocks["A"])
        Be = np.ascontiguousarray(blocks["Be"])
        Ru = np.ascontiguousarray(blocks["R_u"])
        D = np.ascontiguousarray(blocks["D"])
        Rh = np.ascontiguousarray(blocks["R_hat"])
        check(lib.mh_upload_blocks(h, ptr(A), None, ptr(Be), ptr(Ru), ptr(D), ptr(Rh)),
              "mh_upload_blocks")
        fm, ff = C.c_int32(-1), C.c_int32(-1)
        st = lib.mh_factorize(h, C.byref(fm), C.byref(ff), None, None)
        if st == MH_E_SINGULAR_LOCAL:
            raise SingularLocalBlock(plan.e0 + int(fm.value))
        if st == MH_E_SINGULAR_FACE:
            raise SingularFaceBlock(int(plan.owned[int(ff.value)]))
        check(st, "mh_factorize")
        self.f_dev = None
        if self.has_comm or plan.nranks == 1:
            self.f_dev = torch.empty(self.zhat, dtype=torch.float64, device=f"cuda:{device}")
            check(lib.mh_rhs(h, ptr(self.f_dev)), "mh_rhs")

    @property
    def handle(self):
        return self._h.h

    def apply(self, u_dev, w_dev=None):
        torch = _torch()
        w_dev = torch.empty_like(u_dev) if w_dev is None else w_dev
        check(lib.mh_apply(self.handle, ptr(u_dev), ptr(w_dev)), "mh_apply")
        return w_dev

    def gmres(self, tol=1e-10, restart=100, maxiter=10000, precond=True):
        torch = _torch()
        x = torch.empty(self.zhat, dtype=torch.float64, device=f"cuda:{self.device}")
        cap = maxiter + 2
        hist = np.zeros(cap)
        it, conv, hl = C.c_int(0), C.c_int(0), C.c_int(0)
        check(lib.mh_gmres(self.handle, tol, restart, maxiter, 1 if precond else 0, 0,
                           ptr(self.f_dev), ptr(x), C.byref(it), C.byref(conv), ptr(hist), cap,
                           C.byref(hl)), "mh_gmres")
        return x, {"iterations": it.value, "converged": bool(conv.value),
                   "residual_history": hist[:min(hl.value, cap)].tolist()}


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def group_apply(systems: list, u_locals: list) -> list:
    """All ranks of a partition in one process (device-copy transport)."""
    torch = _torch()
    n = len(systems)
    ws = [torch.empty_like(u) for u in u_locals]
    arr = (C.c_void_p * n)(*[s.handle for s in systems])
    ua = (C.c_void_p * n)(*[u.data_ptr() for u in u_locals])
    wa = (C.c_void_p * n)(*[w.data_ptr() for w in ws])
    check(lib.mh_group_apply(arr, n, ua, wa), "mh_group_apply")
    return ws


def local_trace(global_vec: np.ndarray, plan: RankPlan, t: int) -> np.ndarray:
    """The owned part of a global trace vector, in the rank's local order."""
    idx = (plan.owned[:, None] * t + np.arange(t)[None, :]).ravel()
    return np.ascontiguousarray(global_vec[idx])


def scatter_owned(parts: list, plans: list, t: int, zhat: int) -> np.ndarray:
    out = np.full(zhat, np.nan)
    for v, plan in zip(parts, plans):
        idx = (plan.owned[:, None] * t + np.arange(t)[None, :]).ravel()
        out[idx] = v
    return out
