"""Drop-in mirror of ``mehdg.schur_solver`` on the B200 path.

Same names, signatures, error types and report fields as
/root/reference/pkg/src/mehdg/schur_solver.py; the numerics run in
libmehdg_b200.so (hand-written sm_100a CUDA behind a C-ABI), reached through
ctypes.  PyTorch is used only for device buffers and the stream.

  condense              schur_solver.py:185-254  -> mh_upload_* + mh_factorize + mh_rhs
  apply_schur           schur_solver.py:267-293  -> mh_apply   (fused element + face kernels)
  apply_preconditioner  schur_solver.py:296-305  -> mh_precond
  gmres                 schur_solver.py:308-385  -> mh_gmres / mh_gmres_op (device Krylov)
  assemble_schur_explicit schur_solver.py:388-420 -> mh_form_element_schur
  reconstruct_interior  schur_solver.py:423-431  -> mh_reconstruct

Host numpy inputs/outputs behave like the reference; torch CUDA tensors stay
on the device.  There is no CPU fallback: without the library or a GPU these
functions raise.
"""

from __future__ import annotations

import ctypes as C
import functools
import time
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _lib
from ._lib import MH_E_SINGULAR_FACE, MH_E_SINGULAR_LOCAL, MehdgError, check, lib, ptr
from .mesh import condense_tables, mesh_tables


class SingularLocalBlock(RuntimeError):
    """schur_solver.py:33-34 -- carries the macro id."""


class SingularFaceBlock(RuntimeError):
    """schur_solver.py:37-38 -- carries the face id."""


@dataclass
class SolverConfig:
    """schur_solver.py:41-56 (same fields, defaults and validation)."""

    tol: float = 1e-6
    restart: int = 100
    maxiter: int = 10000
    preconditioner: str = "dinv"  # 'dinv' | 'none'
    mode: str = "mf"  # 'mf' | 'mb'
    workers: int = 1
    device: int = 0

    def __post_init__(self):
        if not 0 < self.tol < 1:
            raise ValueError("tolerance must lie in (0, 1)")
        if self.preconditioner not in ("dinv", "none"):
            raise ValueError(f"unknown preconditioner {self.preconditioner!r}")
        if self.mode not in ("mf", "mb"):
            raise ValueError(f"unknown mode {self.mode!r}")


class WorkerPool:
    """schur_solver.py:59-102: a fixed round-robin partition of independent host
    tasks onto threads (item i runs on worker i mod W, so results never depend on
    the worker count), with per-worker thread CPU time for the load-balance
    factor.  On the B200 path the macros and faces are device warps; the pool
    serves host-side callers (e.g. a reference ``assemble_system`` fed to
    ``solve(..., assemble=...)``) and the report's ``lbf`` / ``worker_busy``."""

    def __init__(self, workers: int = 1):
        from concurrent.futures import ThreadPoolExecutor

        self.workers = max(1, int(workers))
        self.busy = np.zeros(self.workers)
        self._ex = ThreadPoolExecutor(max_workers=self.workers) if self.workers > 1 else None

    def map(self, fn: Callable, items) -> list:
        items = list(items)
        out = [None] * len(items)

        def chunk(w):
            t0 = time.thread_time()
            for i in range(w, len(items), self.workers):
                out[i] = fn(items[i])
            self.busy[w] += time.thread_time() - t0

        if self._ex is None:
            chunk(0)
        else:
            for f in [self._ex.submit(chunk, w) for w in range(self.workers)]:
                f.result()
        return out

    @property
    def lbf(self) -> float:
        mx = float(self.busy.max(initial=0.0))
        return 1.0 if mx == 0.0 else float(self.busy.mean()) / mx

    def close(self):
        if self._ex is not None:
            self._ex.shutdown(wait=True)
            self._ex = None


def _torch():
    import torch

    return torch


def _stream_ptr(device: int):
    torch = _torch()
    return torch.cuda.current_stream(device).cuda_stream


class _Handle:
    """Owns one mh_system*."""

    def __init__(self, device, nfe, N, Q, t, F):
        _lib.require_gpu()
        torch = _torch()
        torch.cuda.init()
        self.device = device
        h = C.c_void_p()
        check(lib.mh_create(device, nfe, N, Q, t, F, C.byref(h)), "mh_create")
        self.h = h
        check(lib.mh_set_stream(self.h, _stream_ptr(device)), "mh_set_stream")

    def __del__(self):
        h = getattr(self, "h", None)
        if h and lib is not None:  # lib is None during interpreter shutdown
            lib.mh_destroy(h)
            self.h = None


@dataclass
class CondensedSystem:
    """schur_solver.py:157-182.  Device-resident; the integer tables
    (``offsets``, ``gather_mask``, ``gather_idx``, ``face_plan``) are built on
    first access with the reference's exact semantics."""

    mesh: object
    p: int
    local_ops: Optional[list]
    face_ops: Optional[dict]
    zhat: int
    pool: WorkerPool
    N: int = 0
    Q: int = 0
    t: int = 0
    nfe: int = 3
    F: int = 0
    tables: dict = field(default_factory=dict)
    face_kinds: Optional[np.ndarray] = None
    counters: dict = field(default_factory=lambda: {"macro_apply": 0, "face_reduce": 0})
    timings: dict = field(default_factory=lambda: {"local": 0.0, "global": 0.0})
    _h: Optional[_Handle] = None
    _f_dev: object = None
    _f_host: Optional[np.ndarray] = None
    _offsets: Optional[dict] = None
    _face_ids: Optional[np.ndarray] = None
    _dof_local: int = 0

    # -- reference attributes ------------------------------------------------
    @property
    def handle(self):
        return self._h.h

    @property
    def device(self) -> int:
        return self._h.device

    @property
    def nc(self) -> int:
        return self.nfe * self.t

    @property
    def dof_local(self) -> int:
        return self._dof_local

    @property
    def f_vec(self) -> np.ndarray:
        if self._f_host is None:
            self._f_host = self.f_device.cpu().numpy()
        return self._f_host

    @property
    def f_device(self):
        return self._f_dev

    @property
    def face_ids(self) -> np.ndarray:
        """Skeleton face id of each unknown face, in trace order."""
        if self._face_ids is None:
            self._face_ids = np.nonzero(self.tables["uidx"] >= 0)[0]
        return self._face_ids

    @property
    def offsets(self) -> dict:
        if self._offsets is None:
            self._offsets = {int(fid): (u * self.t, self.t) for u, fid in enumerate(self.face_ids)}
        return self._offsets

    @property
    def gather_mask(self) -> list:
        ef = self.tables["elem_ufac"]
        t = self.t
        return [np.repeat(ef[e] >= 0, t) for e in range(self.N)]

    @property
    def gather_idx(self) -> list:
        ef = self.tables["elem_ufac"]
        t = self.t
        out = []
        for e in range(self.N):
            u = ef[e][ef[e] >= 0].astype(np.int64)
            out.append((u[:, None] * t + np.arange(t)[None, :]).ravel())
        return out

    @property
    def face_plan(self) -> list:
        fe, fs = self.tables["face_elem"], self.tables["face_slot"]
        t = self.t
        plan = []
        for u, fid in enumerate(self.face_ids):
            order = [(int(fe[u, c]), slice(int(fs[u, c]) * t, (int(fs[u, c]) + 1) * t))
                     for c in range(2) if fe[u, c] >= 0]
            plan.append((int(fid), u * t, t, order))
        return plan

    def gather(self, uhat: np.ndarray, e: int) -> np.ndarray:
        ue = np.zeros(self.nc)
        ue[self.gather_mask[e]] = np.asarray(uhat)[self.gather_idx[e]]
        return ue


# ---------------------------------------------------------------------------
# the factors the reference stores in its operator objects

class _DeviceLU:
    """``op.lu`` of a condensed macro: ``("dense", (lu, piv))`` in scipy's layout,
    fetched from the device on first access (the reference stores it at
    condense, schur_solver.py:111)."""

    __slots__ = ("_sys", "_e", "_val")

    def __init__(self, sys, e):
        self._sys, self._e, self._val = sys, e, None

    def _get(self):
        if self._val is None:
            lu, piv = local_factors(self._sys, self._e, 1)
            self._val = ("dense", (lu[0], piv[0]))
        return self._val

    def __getitem__(self, i):
        return self._get()[i]

    def __len__(self):
        return 2

    def __iter__(self):
        return iter(self._get())

    def __repr__(self):
        return f"_DeviceLU(macro={self._e})"


class _DeviceFaceFactor:
    """``op.factor`` of a condensed face: ``("inv", 1.0, D^-1)`` -- the explicit
    inverse the device preconditioner applies (sign folded in) -- fetched on
    first access.  Replacing ``op.factor`` after condense (as the reference's
    tests do, test_schur_solver.py:138-147) is honoured by
    ``apply_preconditioner``: the replaced faces' inverses are recomputed from
    the new factor with the reference's solve rule and uploaded."""

    __slots__ = ("_sys", "_u", "_val")

    def __init__(self, sys, u):
        self._sys, self._u, self._val = sys, u, None

    def _get(self):
        if self._val is None:
            t = self._sys.t
            inv = np.empty((1, t, t))
            check(lib.mh_get_face_inverse(self._sys.handle, 1, ptr(np.array([self._u], np.int32)),
                                          ptr(inv)), "mh_get_face_inverse")
            self._val = ("inv", 1.0, inv[0])
        return self._val

    def __getitem__(self, i):
        return self._get()[i]

    def __len__(self):
        return 3

    def __iter__(self):
        return iter(self._get())

    def __repr__(self):
        return f"_DeviceFaceFactor(face={self._u})"


def _face_inverse_from_factor(factor, t):
    """D^-1 (sign folded in) from a reference face factor (schur_solver.py:150-154)."""
    import scipy.linalg as sla

    kind, sign, fac = factor
    eye = np.eye(t)
    if kind == "chol":
        return sign * sla.cho_solve(fac, eye)
    if kind == "inv":
        return sign * np.asarray(fac)
    return sla.lu_solve(fac, eye)


def _sync_face_factors(sys) -> None:
    """Upload the inverses of faces whose ``op.factor`` was replaced since condense."""
    if sys.face_ops is None:
        return
    idx, inv = [], []
    for u, fid in enumerate(sys.face_ids):
        fop = sys.face_ops[int(fid)]
        fac = getattr(fop, "factor", None)
        if isinstance(fac, _DeviceFaceFactor) and fac._sys is sys:
            continue
        idx.append(u)
        inv.append(_face_inverse_from_factor(fac, sys.t))
        fop.factor = _DeviceFaceFactor(sys, u)
        fop.factor._val = ("inv", 1.0, inv[-1])
    if idx:
        arr = np.ascontiguousarray(np.stack(inv))
        check(lib.mh_set_face_inverse(sys.handle, len(idx), ptr(np.asarray(idx, np.int32)),
                                      ptr(arr)), "mh_set_face_inverse")


# ---------------------------------------------------------------------------
# condense

def _stack_ops(local_ops: list, face_ops: dict, tables: dict):
    """Stack LocalOperators / FaceOperator blocks into the C-ABI layouts,
    checking the slot layout of assemble_macro (assembly.py:241-249): slot k of a
    macro owns columns [k t, (k+1) t); macros with fewer faces than the widest
    one (2:1 hanging faces) are padded with empty slots."""
    N = len(local_ops)
    op0 = local_ops[0]
    nloc = int(op0.R_u.size)
    nfe = tables["nfe"]
    sl0 = op0.face_slots[0][1]
    t = int(sl0.stop - sl0.start)
    nc = nfe * t
    A = np.empty((N, nloc, nloc))
    B = np.zeros((N, nloc, nc))
    Cm = np.zeros((N, nc, nloc))
    Ru = np.empty((N, nloc))
    c_is_bt = True
    for e, op in enumerate(local_ops):
        if op.macro_id != e:
            raise ValueError("local_ops must be ordered by macro id")
        a = op.A.toarray() if hasattr(op.A, "toarray") else np.asarray(op.A)
        nce = len(op.face_slots) * t
        if a.shape != (nloc, nloc) or op.B.shape != (nloc, nce) or op.C.shape != (nce, nloc) \
                or nce > nc:
            raise NotImplementedError("all macros must share one block size and slot width")
        for k, (fid, sl) in enumerate(op.face_slots):
            if sl.start != k * t or sl.stop != (k + 1) * t:
                raise NotImplementedError("face slot k must own columns [k t, (k+1) t)")
            if tables["elem_face"][e, k] != fid:
                raise ValueError("face_slots disagree with the mesh skeleton")
        A[e] = a
        B[e, :, :nce] = op.B
        Cm[e, :nce] = op.C
        Ru[e] = op.R_u
        if c_is_bt and not np.array_equal(op.C, op.B.T):
            c_is_bt = False
    uidx = tables["uidx"]
    F = int((uidx >= 0).sum())
    D = np.empty((F, t, t))
    Rh = np.empty((F, t))
    for fid in np.nonzero(uidx >= 0)[0]:
        fop = face_ops[int(fid)]
        D[uidx[fid]] = fop.D
        Rh[uidx[fid]] = fop.R_hat
    return A, B, (None if c_is_bt else Cm), Ru, D, Rh, nloc, t


def condense_arrays(mesh, A, B, Cm, R_u, D, R_hat, config: SolverConfig, *, p: int = 0,
                    tables: Optional[dict] = None, local_ops=None, face_ops=None,
                    device: Optional[int] = None, pool: Optional[WorkerPool] = None,
                    b_is_ct: bool = False) -> CondensedSystem:
    """Upload stacked blocks and factorise them on the device.

    A (N,Q,Q); B (N,Q,nc) = op.B or None; Cm (N,nc,Q) = op.C or None (None means
    op.C = op.B^T, resp. op.B = op.C^T -- the synthetic operator); R_u (N,Q);
    D (F,t,t), R_hat (F,t) in unknown-face order."""
    if tables is None:
        tables = mesh_tables(mesh)
        tables.update(condense_tables(tables))
    tables = dict(tables)
    on_device = _is_torch(A)
    if face_ops is None:  # host face blocks for assemble_schur_explicit
        tables["D"] = D.detach().cpu().numpy() if on_device else D
    N, Q = A.shape[0], A.shape[1]
    nfe = tables["nfe"]
    F = int(tables["F"]) if "F" in tables else int((tables["uidx"] >= 0).sum())
    t = D.shape[1] if D.shape[0] else ((B.shape[2] if B is not None else Cm.shape[1]) // nfe)
    dev = config.device if device is None else device
    torch = _torch()
    h = _Handle(dev, nfe, N, Q, t, F)
    check(lib.mh_upload_connectivity(h.h, ptr(np.ascontiguousarray(tables["elem_ufac"], np.int32)),
                                     ptr(np.ascontiguousarray(tables["face_elem"], np.int32)),
                                     ptr(np.ascontiguousarray(tables["face_slot"], np.int32))),
          "mh_upload_connectivity")

    if on_device:  # blocks assembled on the device (assemble_system_device)
        def dp(x):
            return None if x is None else x.contiguous().data_ptr()

        keep = [x.contiguous() if x is not None else None for x in (A, B, Cm, R_u, D, R_hat)]
        check(lib.mh_upload_blocks_device(h.h, *[dp(x) for x in keep]), "mh_upload_blocks_device")
        torch.cuda.current_stream(dev).synchronize()
    else:
        def c64(x):
            return None if x is None else np.ascontiguousarray(x, dtype=np.float64)

        A_, B_, C_, Ru_, D_, Rh_ = c64(A), c64(B), c64(Cm), c64(R_u), c64(D), c64(R_hat)
        check(lib.mh_upload_blocks(h.h, ptr(A_), ptr(B_), ptr(C_), ptr(Ru_), ptr(D_), ptr(Rh_)),
              "mh_upload_blocks")
    fm, ff = C.c_int32(-1), C.c_int32(-1)
    kinds = np.empty(F, np.int8)
    lu_ms = C.c_float(0.0)
    t0 = time.perf_counter()
    st = lib.mh_factorize(h.h, C.byref(fm), C.byref(ff), ptr(kinds), C.byref(lu_ms))
    if st == MH_E_SINGULAR_LOCAL:
        raise SingularLocalBlock(int(fm.value))
    if st == MH_E_SINGULAR_FACE:
        raise SingularFaceBlock(int(ff.value))
    check(st, "mh_factorize")
    f_dev = torch.empty(F * t, dtype=torch.float64, device=f"cuda:{dev}")
    check(lib.mh_rhs(h.h, ptr(f_dev)), "mh_rhs")
    torch.cuda.current_stream(dev).synchronize()
    sys = CondensedSystem(mesh=mesh, p=p, local_ops=local_ops, face_ops=face_ops, zhat=F * t,
                          pool=pool or WorkerPool(config.workers), N=N, Q=Q, t=t, nfe=nfe, F=F,
                          tables=tables, face_kinds=kinds, _h=h, _f_dev=f_dev,
                          _dof_local=N * Q)
    sys.timings["factorize"] = time.perf_counter() - t0
    sys.timings["lu_kernel_ms"] = float(lu_ms.value)
    if face_ops is not None:
        names = _lib.FACE_KIND_NAMES
        for fid, u in zip(sys.face_ids, range(F)):
            fop = face_ops[int(fid)]
            fop.factor_kind = names[int(kinds[u])]
    return sys


def condense(mesh, local_ops: list, face_ops: dict, config: SolverConfig,
             pool: Optional[WorkerPool] = None, host_factors: bool = False) -> CondensedSystem:
    """schur_solver.py:185-254: factorise every block on the device and form
    f = R_hat - sum C A^-1 R_u.

    The reference stores scipy factors in ``op.lu`` / ``op.factor`` (mutating
    its inputs, schur_solver.py:111, 137-147).  Here the factors stay on the
    device; ``host_factors=True`` copies them back into those fields in the
    reference's layout (``("dense", (lu, piv))``; faces ``("inv", 1.0, D^-1)``)."""
    tables = mesh_tables(mesh)
    tables.update(condense_tables(tables))
    A, B, Cm, Ru, D, Rh, nloc, t = _stack_ops(local_ops, face_ops, tables)
    m = mesh.macro_elements[0].m if len(mesh.macro_elements) else 1
    sys = condense_arrays(mesh, A, B, Cm, Ru, D, Rh, config, p=_infer_p(nloc, m),
                          tables=tables, local_ops=local_ops, face_ops=face_ops, pool=pool)
    # the reference's in-place factor fields (schur_solver.py:111, 137-147):
    # device-backed, fetched on access; host_factors=True fetches them now
    if host_factors:
        lu, piv = local_factors(sys)
        for e, op in enumerate(local_ops):
            op.lu = ("dense", (lu[e], piv[e]))
    else:
        for e, op in enumerate(local_ops):
            op.lu = _DeviceLU(sys, e)
    for u, fid in enumerate(sys.face_ids):
        face_ops[int(fid)].factor = _DeviceFaceFactor(sys, u)
    return sys


def _infer_p(nloc: int, m: int) -> int:
    """schur_solver.py:257-264 (meaningful only for real 3Q-sized blocks)."""
    from math import isqrt

    Q = nloc // 3
    L = (isqrt(8 * Q + 1) - 3) // 2
    return L // m


# ---------------------------------------------------------------------------
# operator

def _is_torch(x) -> bool:
    return hasattr(x, "data_ptr") and hasattr(x, "is_cuda")


def _dev_vec(sys, n=None):
    torch = _torch()
    return torch.empty(sys.zhat if n is None else n, dtype=torch.float64,
                       device=f"cuda:{sys.device}")


def _run(sys, fn, name, x, out=None):
    """Apply a device op to numpy (host path) or torch CUDA input.  `out`
    (optional) receives the result -- e.g. a pinned host array."""
    if _is_torch(x):
        if x.dtype != _torch().float64 or not x.is_cuda:
            raise TypeError("device vectors must be float64 CUDA tensors")
        x = x.contiguous()
        out = _dev_vec(sys) if out is None else out
        check(fn(sys.handle, ptr(x), ptr(out)), name)
        return out
    xh = np.ascontiguousarray(x, dtype=np.float64)
    if xh.shape != (sys.zhat,):
        raise ValueError(f"expected a vector of length {sys.zhat}")
    if out is None:
        out = np.empty(sys.zhat)
    elif out.shape != (sys.zhat,) or out.dtype != np.float64 or not out.flags.c_contiguous:
        raise ValueError("out must be a contiguous float64 vector of length zhat")
    host_fn = {"mh_apply": lib.mh_apply_host, "mh_precond": lib.mh_precond_host}[name]
    check(host_fn(sys.handle, ptr(xh), ptr(out)), name)
    return out


def apply_schur(sys: CondensedSystem, uhat, out=None):
    """(D - C A^-1 B) uhat via the fused element kernel + face reduction
    (schur_solver.py:267-293).  ``out`` is an optional preallocated result
    (numpy for host input -- pinned memory avoids a staged copy -- or a CUDA
    tensor for device input); the reference signature is the default."""
    t0 = time.perf_counter()
    w = _run(sys, lib.mh_apply, "mh_apply", uhat, out)
    sys.counters["macro_apply"] += sys.N
    sys.counters["face_reduce"] += sys.F
    sys.timings["local"] += time.perf_counter() - t0
    return w


def apply_schur_many(sys: CondensedSystem, U, out=None, repeat: Optional[int] = None):
    """The operator on a stack of host vectors U (k x zhat numpy), returning
    W (k x zhat): the host->device copy of vector i+1 and the device->host copy
    of vector i-1 overlap the apply of vector i (mh_apply_host_many).  With
    ``repeat=k`` a single vector U (zhat,) is applied k times into one output
    (k copies in and out, as a streaming benchmark does).  Pinned host
    memory (e.g. ``torch.empty(..., pin_memory=True).numpy()``) keeps the
    copies asynchronous."""
    U = np.asarray(U)
    if U.dtype != np.float64 or not U.flags.c_contiguous:
        raise ValueError("U must be a contiguous float64 array")
    if repeat is not None:
        if U.shape != (sys.zhat,):
            raise ValueError(f"expected a vector of length {sys.zhat} with repeat=")
        k, ldu = int(repeat), 0
        shape = (sys.zhat,)
    else:
        if U.ndim != 2 or U.shape[1] != sys.zhat:
            raise ValueError(f"expected a (k, {sys.zhat}) array")
        k, ldu = U.shape[0], sys.zhat
        shape = U.shape
    if out is None:
        out = np.empty(shape)
    elif out.shape != shape or out.dtype != np.float64 or not out.flags.c_contiguous:
        raise ValueError(f"out must be a contiguous float64 array of shape {shape}")
    t0 = time.perf_counter()
    check(lib.mh_apply_host_many(sys.handle, k, ptr(U), ldu, ptr(out),
                                 0 if repeat is not None else sys.zhat), "mh_apply_host_many")
    sys.counters["macro_apply"] += k * sys.N
    sys.counters["face_reduce"] += k * sys.F
    sys.timings["local"] += time.perf_counter() - t0
    return out


def apply_preconditioner(sys: CondensedSystem, w):
    """Per-face D^-1 (schur_solver.py:296-305), with the face factors in
    ``sys.face_ops`` -- including ones replaced after condense."""
    _sync_face_factors(sys)
    return _run(sys, lib.mh_precond, "mh_precond", w)


class SchurOperator:
    """``lambda v: apply_schur(sys, v)`` that gmres recognises and runs
    entirely on the device (mode 'mf', or 'mb' after assemble_schur_explicit)."""

    def __init__(self, sys: CondensedSystem, mode: str = "mf"):
        self.sys, self.mode = sys, mode

    def __call__(self, v):
        if self.mode == "mb":
            return apply_schur_mb(self.sys, v)
        return apply_schur(self.sys, v)


class Preconditioner:
    """``lambda w: apply_preconditioner(sys, w)`` recognised by gmres."""

    def __init__(self, sys: CondensedSystem):
        self.sys = sys

    def __call__(self, w):
        return apply_preconditioner(self.sys, w)


def _bound_system(op, kind):
    if kind == "A" and isinstance(op, SchurOperator):
        return op.sys, op.mode
    if kind == "M" and isinstance(op, Preconditioner):
        return op.sys, None
    if isinstance(op, functools.partial) and op.args and isinstance(op.args[0], CondensedSystem):
        if kind == "A" and op.func is apply_schur:
            return op.args[0], "mf"
        if kind == "M" and op.func is apply_preconditioner:
            return op.args[0], None
    return None, None


def gmres(apply_op: Callable, rhs, config: SolverConfig, precond: Optional[Callable] = None):
    """Restarted left-preconditioned GMRES (schur_solver.py:308-385) on the device.

    Returns (x, info) with info = {iterations, residual_history, converged}.
    A SchurOperator / Preconditioner pair runs without any Python per
    iteration; other callables are called back with numpy vectors (numpy rhs)
    or CUDA tensors (tensor rhs)."""
    torch = _torch()
    sysA, mode = _bound_system(apply_op, "A")
    sysM, _ = _bound_system(precond, "M") if precond is not None else (None, None)
    if sysM is not None:
        _sync_face_factors(sysM)
    host = not _is_torch(rhs)
    n = int(rhs.numel() if not host else np.asarray(rhs).size)
    cap = config.maxiter + 2
    hist = np.zeros(cap)
    it, conv, hl = C.c_int(0), C.c_int(0), C.c_int(0)
    if sysA is not None and (precond is None or sysM is sysA):
        sys = sysA
        r = torch.as_tensor(np.ascontiguousarray(rhs, np.float64), device=f"cuda:{sys.device}") \
            if host else rhs.contiguous()
        x = _dev_vec(sys)
        t0 = time.perf_counter()
        check(lib.mh_gmres(sys.handle, config.tol, config.restart, config.maxiter,
                           1 if precond is not None else 0, 1 if mode == "mb" else 0,
                           ptr(r), ptr(x), C.byref(it), C.byref(conv), ptr(hist), cap,
                           C.byref(hl)), "mh_gmres")
        sys.timings["gmres"] = time.perf_counter() - t0
    else:
        _lib.require_gpu()
        dev = torch.cuda.current_device()
        r = torch.as_tensor(np.ascontiguousarray(rhs, np.float64), device=f"cuda:{dev}") \
            if host else rhs.contiguous()
        x = torch.empty(n, dtype=torch.float64, device=r.device)
        errors = []

        def wrap(fn):
            def cb(ctx, pin, pout):
                try:
                    vin = _wrap_dev(pin, n, r.device)
                    vout = _wrap_dev(pout, n, r.device)
                    if host:
                        res = np.asarray(fn(vin.cpu().numpy()), dtype=np.float64)
                        vout.copy_(torch.from_numpy(np.ascontiguousarray(res)))
                    else:
                        vout.copy_(fn(vin))
                    return 0
                except BaseException as exc:  # reported after the C call returns
                    errors.append(exc)
                    return _lib.MH_E_CALLBACK
            return _lib.OP_FN(cb)

        cbA = wrap(apply_op)
        cbM = wrap(precond) if precond is not None else C.cast(None, _lib.OP_FN)
        st = lib.mh_gmres_op(r.device.index or 0, _stream_ptr(r.device.index or 0), n, cbA, None,
                             cbM, None, config.tol, config.restart, config.maxiter, ptr(r),
                             ptr(x), C.byref(it), C.byref(conv), ptr(hist), cap, C.byref(hl))
        if errors:
            raise errors[0]
        check(st, "mh_gmres_op")
    torch.cuda.current_stream(x.device).synchronize()
    info = {"iterations": int(it.value), "residual_history": hist[:min(hl.value, cap)].tolist(),
            "converged": bool(conv.value)}
    return (x.cpu().numpy() if host else x), info


class _CudaView:
    def __init__(self, p, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (p, False),
                                         "version": 3, "strides": None}


def _wrap_dev(p, n, device):
    return _torch().as_tensor(_CudaView(p, n), device=device)


def reconstruct_interior(sys: CondensedSystem, uhat) -> list:
    """Per macro u_e = A^-1 (R_u - B gather(uhat)) (schur_solver.py:423-431).
    Returns a list of per-macro arrays for numpy input, an (N, Q) tensor for
    CUDA input."""
    torch = _torch()
    if _is_torch(uhat):
        U = torch.empty((sys.N, sys.Q), dtype=torch.float64, device=uhat.device)
        check(lib.mh_reconstruct(sys.handle, ptr(uhat.contiguous()), ptr(U)), "mh_reconstruct")
        return U
    u = np.ascontiguousarray(uhat, np.float64)
    U = np.empty((sys.N, sys.Q))
    check(lib.mh_reconstruct_host(sys.handle, ptr(u), ptr(U)), "mh_reconstruct")
    return list(U)


def form_element_schur(sys: CondensedSystem) -> None:
    check(lib.mh_form_element_schur(sys.handle), "mh_form_element_schur")


def apply_schur_mb(sys: CondensedSystem, uhat):
    return _run_mb(sys, uhat)


def _run_mb(sys, x):
    if _is_torch(x):
        out = _dev_vec(sys)
        check(lib.mh_apply_mb(sys.handle, ptr(x.contiguous()), ptr(out)), "mh_apply_mb")
        return out
    torch = _torch()
    xd = torch.as_tensor(np.ascontiguousarray(x, np.float64), device=f"cuda:{sys.device}")
    out = _dev_vec(sys)
    check(lib.mh_apply_mb(sys.handle, ptr(xd), ptr(out)), "mh_apply_mb")
    return out.cpu().numpy()


def assemble_schur_explicit(sys: CondensedSystem):
    """Explicit D - C A^-1 B as scipy CSR (schur_solver.py:388-420); the
    element blocks are formed on the device."""
    import scipy.sparse as sp

    form_element_schur(sys)
    nc, t = sys.nc, sys.t
    blocks = np.empty((sys.N, nc, nc))
    check(lib.mh_get_element_schur(sys.handle, 0, sys.N, ptr(blocks)), "mh_get_element_schur")
    ef = sys.tables["elem_ufac"]
    rows, cols, vals = [], [], []
    for e in range(sys.N):
        mask = np.repeat(ef[e] >= 0, t)
        if not mask.any():
            continue
        u = ef[e][ef[e] >= 0].astype(np.int64)
        gi = (u[:, None] * t + np.arange(t)[None, :]).ravel()
        R, Cc = np.meshgrid(gi, gi, indexing="ij")
        rows.append(R.ravel())
        cols.append(Cc.ravel())
        vals.append(blocks[e][np.ix_(mask, mask)].ravel())
    Dh = face_blocks(sys)
    for u in range(sys.F):
        gi = np.arange(u * t, (u + 1) * t)
        R, Cc = np.meshgrid(gi, gi, indexing="ij")
        rows.append(R.ravel())
        cols.append(Cc.ravel())
        vals.append(Dh[u].ravel())
    S = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(sys.zhat, sys.zhat))
    return S.tocsr()


def face_blocks(sys: CondensedSystem) -> np.ndarray:
    """The F face blocks D (unknown-face order) -- from the host ops if given."""
    if sys.face_ops is not None:
        return np.stack([sys.face_ops[int(fid)].D for fid in sys.face_ids]) if sys.F else \
            np.zeros((0, sys.t, sys.t))
    if "D" in sys.tables:
        return sys.tables["D"]
    raise ValueError("face blocks are not kept on the host for array-condensed systems")


def local_factors(sys: CondensedSystem, first: int = 0, count: Optional[int] = None):
    """Packed L\\U (row-major, scipy layout) and 0-based LAPACK pivots."""
    count = sys.N - first if count is None else count
    lu = np.empty((count, sys.Q, sys.Q))
    piv = np.empty((count, sys.Q), np.int32)
    check(lib.mh_get_local_factors(sys.handle, first, count, ptr(lu), ptr(piv)),
          "mh_get_local_factors")
    return lu, piv


# ---------------------------------------------------------------------------
# reports and the solve driver

@dataclass
class SolveReport:
    """schur_solver.py:434-462."""

    p: int
    m: int
    n: int
    dof_local: int
    dof_global: int
    iterations: int
    converged: bool
    tol: float
    mode: str
    precond: str
    t_init_s: float
    t_local_s: float
    t_global_s: float
    t_reconstruct_s: float
    lbf: float
    worker_busy: list
    residual_history: list

    def to_record(self) -> dict:
        return {
            "p": self.p, "m": self.m, "n": self.n,
            "dof_local": self.dof_local, "dof_global": self.dof_global,
            "iterations": self.iterations, "converged": self.converged,
            "tol": self.tol, "mode": self.mode, "precond": self.precond,
            "t_init_s": self.t_init_s, "t_local_s": self.t_local_s,
            "t_global_s": self.t_global_s, "lbf": self.lbf,
        }


@dataclass
class Solution:
    """schur_solver.py:465-479."""

    local: list
    uhat: np.ndarray
    report: SolveReport

    def u_coeffs(self, e: int) -> np.ndarray:
        v = self.local[e]
        Q = v.size // 3
        return v[2 * Q:]

    def q_coeffs(self, e: int) -> np.ndarray:
        v = self.local[e]
        Q = v.size // 3
        return v[:2 * Q].reshape(2, Q)


def solve_condensed(sys: CondensedSystem, config: SolverConfig, t_init: float = 0.0):
    """The post-assembly half of ``solve`` (schur_solver.py:506-541)."""
    precond = Preconditioner(sys) if config.preconditioner == "dinv" else None
    if config.mode == "mb":
        form_element_schur(sys)
    op = SchurOperator(sys, config.mode)
    # t_local: the element kernels' time inside the solve (CUDA events around
    # each launch, mh_profile) -- the reference sums its local tasks' time the
    # same way (schur_solver.py:518-535); t_global is the rest of GMRES
    h = sys.handle
    check(lib.mh_profile_read(h, None, None, None, None), "profile")
    check(lib.mh_profile(h, 1), "profile")
    t0 = time.perf_counter()
    try:
        uhat, info = gmres(op, sys.f_device, config, precond=precond)
    finally:
        t_gmres = time.perf_counter() - t0
        ems = C.c_double()
        check(lib.mh_profile_read(h, C.byref(ems), None, None, None), "profile")
        check(lib.mh_profile(h, 0), "profile")
    t_local = ems.value / 1e3
    sys.timings["local"] = t_local
    t0 = time.perf_counter()
    U = reconstruct_interior(sys, uhat)
    local = list(U.cpu().numpy())
    t_rec = time.perf_counter() - t0
    mesh = sys.mesh
    report = SolveReport(
        p=sys.p, m=mesh.macro_elements[0].m if len(mesh.macro_elements) else 0,
        n=getattr(mesh, "n", 0), dof_local=sys.dof_local, dof_global=sys.zhat,
        iterations=info["iterations"], converged=info["converged"], tol=config.tol,
        mode=config.mode, precond=config.preconditioner, t_init_s=t_init,
        t_local_s=t_local, t_global_s=max(t_gmres - t_local, 0.0), t_reconstruct_s=t_rec,
        lbf=sys.pool.lbf,
        worker_busy=list(sys.pool.busy), residual_history=info["residual_history"])
    return Solution(local=local, uhat=uhat.cpu().numpy(), report=report), sys


def solve(mesh, problem, stab, config: SolverConfig, p: int, assemble: Optional[Callable] = None):
    """schur_solver.py:495-541: assemble, condense, GMRES on the trace system,
    reconstruct.  By default the blocks are assembled on the device
    (assembly.assemble_system_device, 2-D) and never leave it; a callable
    ``assemble(mesh, problem, stab, p) -> (local_ops, face_ops)`` (e.g. the
    reference's ``assemble_system``) takes the host path instead."""
    if assemble is None:
        from .assembly import assemble_system_device

        t0 = time.perf_counter()
        blk = assemble_system_device(mesh, problem, stab, p, device=config.device)
        t_asm = time.perf_counter() - t0
        t0 = time.perf_counter()
        sys = condense_arrays(mesh, blk.A, blk.B, blk.C, blk.R_u, blk.D, blk.R_hat, config,
                              p=p, tables=blk.tables)
        sys.timings["assemble"] = t_asm
        return solve_condensed(sys, config, t_init=time.perf_counter() - t0)
    local_ops, face_ops = assemble(mesh, problem, stab, p)
    t0 = time.perf_counter()
    sys = condense(mesh, local_ops, face_ops, config)
    return solve_condensed(sys, config, t_init=time.perf_counter() - t0)
