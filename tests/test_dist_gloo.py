"""Multi-rank path on CPU: world_size-2 (and 3) gloo process groups run the
slab halo choreography of the NCCL path -- uhat halo, per-macro element
contributions, v return to the face owner, left-then-right face reduction,
rank-ordered dot products -- with the oracle's per-macro arithmetic, and the
assembled result must equal the single-rank oracle apply bit for bit."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import scipy.linalg as sla
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import solver_oracle as SO
from paper_2302_10917_b200 import synthetic as S
from paper_2302_10917_b200.partition import partition, rank_plan

CASES = [(2, 4, 2, 2), (3, 2, 1, 3), (2, 5, 1, 3)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_apply(prob, plan, u_global):
    """One rank's apply, exchanging through the default (gloo) group."""
    t, nfe = prob["t"], prob["d"] + 1
    me, nr = plan.rank, plan.nranks
    u_own = u_global[(plan.owned[:, None] * t + np.arange(t)).ravel()]
    # 1. uhat halo: owners send, neighbours receive (grouped by peer)
    reqs, recv = [], []
    off = 0
    for q in range(nr):
        c = int(plan.send_count[q])
        if c:
            seg = u_own.reshape(-1, t)[plan.send_face[off:off + c]].ravel()
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(seg)), q))
        off += c
    for q in range(nr):
        c = int(plan.recv_count[q])
        buf = torch.empty(c * t, dtype=torch.float64)
        if c:
            reqs.append(dist.irecv(buf, q))
        recv.append(buf)
    for r in reqs:
        r.wait()
    u_loc = np.concatenate([u_own] + [b.numpy() for b in recv])
    # 2. element contributions of the local macros (oracle arithmetic)
    n_loc = plan.n_local
    V = np.zeros((n_loc * nfe + int(plan.vrecv_count.sum())) * t)
    for el in range(n_loc):
        e = plan.e0 + el
        ue = np.zeros(nfe * t)
        for k in range(nfe):
            f = plan.elem_ufac[el, k]
            if f >= 0:
                ue[k * t:(k + 1) * t] = u_loc[f * t:(f + 1) * t]
        lu = sla.lu_factor(prob["A"][e])
        y = sla.lu_solve(lu, prob["B"][e] @ ue)
        V[el * nfe * t:(el + 1) * nfe * t] = prob["C"][e] @ y
    # 3. v return to the face owners
    reqs, off, roff = [], 0, n_loc * nfe * t
    vseg = V[:n_loc * nfe * t].reshape(-1, t)
    for q in range(nr):
        c = int(plan.vret_count[q])
        if c:
            seg = vseg[plan.vret_slot[off:off + c]].ravel()
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(seg)), q))
        off += c
    bufs = []
    for q in range(nr):
        c = int(plan.vrecv_count[q])
        if c:
            b = torch.empty(c * t, dtype=torch.float64)
            reqs.append(dist.irecv(b, q))
            bufs.append((roff, b))
        roff += c * t
    for r in reqs:
        r.wait()
    for o, b in bufs:
        V[o:o + b.numel()] = b.numpy()
    # 4. face reduction on owned faces: left first, then right
    w = np.empty(plan.F_own * t)
    for lf, gf in enumerate(plan.owned):
        seg = prob["D"][gf] @ u_own[lf * t:(lf + 1) * t]
        for c in range(2):
            el = plan.face_elem[lf, c]
            if el < 0:
                continue
            slot = el * nfe + plan.face_slot[lf, c] if el < n_loc else n_loc * nfe + (el - n_loc)
            seg = seg - V[slot * t:(slot + 1) * t]
        w[lf * t:(lf + 1) * t] = seg
    return w


def _worker(rank, world, port, case, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d, n, m, p = case
        prob = S.make_problem(d, n, m, p, seed=5)
        eb = partition(d, n, prob["N"], world)
        plan = rank_plan(prob["elem_face"], prob["face_elem"], prob["face_slot"], eb, rank)
        w = _rank_apply(prob, plan, prob["uhat"])
        # rank-ordered dot product (the Krylov reduction of the NCCL path)
        local = float(w @ w)
        parts = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.tensor([local], dtype=torch.float64))
        total = 0.0
        for pt in parts:
            total += float(pt.item())
        out_q.put((rank, plan.owned.tolist(), w.tolist(), total))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", CASES)
def test_gloo_slab_apply_is_bitwise_single_rank(world, case):
    d, n, m, p = case
    prob = S.make_problem(d, n, m, p, seed=5)
    o = SO.system_from_problem(prob).factorize()
    w_ref = o.apply(prob["uhat"])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    t = prob["t"]
    w = np.full(prob["zhat"], np.nan)
    totals = set()
    for rank, owned, wl, total in res:
        owned = np.asarray(owned, np.int64)
        w[(owned[:, None] * t + np.arange(t)).ravel()] = wl
        totals.add(total)
    assert not np.isnan(w).any()
    assert np.array_equal(w, w_ref)
    assert len(totals) == 1  # every rank sums the partials in the same order
    assert abs(totals.pop() - float(w_ref @ w_ref)) <= 1e-12 * float(w_ref @ w_ref)


@pytest.mark.parametrize("case", CASES + [(2, 16, 1, 1), (3, 4, 1, 1)])
@pytest.mark.parametrize("world", [2, 3, 4])
def test_rank_plans_cover_every_face_once(case, world):
    d, n, m, p = case
    prob = S.make_problem(d, n, m, p, with_blocks=False)
    eb = partition(d, n, prob["N"], world)
    plans = [rank_plan(prob["elem_face"], prob["face_elem"], prob["face_slot"], eb, r)
             for r in range(world)]
    owned = np.concatenate([pl.owned for pl in plans])
    assert np.array_equal(np.sort(owned), np.arange(prob["F"]))
    for pl in plans:
        # halo faces of rank r are owned by lower ranks; sends match receives
        for q in range(world):
            other = plans[q]
            assert other.send_count[pl.rank] == pl.recv_count[q]
            assert pl.vret_count[q] == other.vrecv_count[pl.rank]
        assert pl.elem_ufac.max(initial=-1) < pl.F_own + pl.F_halo
    if d == 2 and eb[1] % (2 * n) == 0:
        # whole mesh rows: each slab interface carries exactly n faces
        assert plans[0].send_count[1] == n
    if d == 3 and eb[1] % (6 * n * n) == 0:
        assert plans[0].send_count[1] == 2 * n * n
