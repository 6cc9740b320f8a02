"""Slab-partitioned operator on ONE GPU: every rank of a partition is a
separate mh_system with its halo plan, the exchanges are device copies
(mh_group_apply).  The device halo kernels, extra v-slots and face tables
must reproduce the single-system apply bit for bit (the NCCL path runs the
same phases with ncclSend/ncclRecv)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2302_10917_b200 as P
from paper_2302_10917_b200 import synthetic as S
from paper_2302_10917_b200.distributed import RankSystem, group_apply, local_trace, nccl_unique_id
from paper_2302_10917_b200.partition import partition, rank_plan

pytestmark = pytest.mark.gpu


def single_system(prob):
    tables = {"nfe": prob["d"] + 1, "elem_ufac": prob["elem_face"],
              "face_elem": prob["face_elem"], "face_slot": prob["face_slot"],
              "uidx": prob["uidx"], "F": prob["F"]}
    return P.condense_arrays(prob["mesh"], prob["A"], None, prob["Be"], prob["R_u"], prob["D"],
                             prob["R_hat"], P.SolverConfig(tol=1e-10), tables=tables)


@pytest.mark.parametrize("case,world", [((2, 8, 2, 2), 2), ((2, 8, 2, 2), 4), ((3, 4, 1, 3), 2),
                                        ((3, 3, 2, 2), 3), ((2, 16, 2, 3), 8)])
def test_group_apply_bitwise_equals_single(gpu, case, world):
    d, n, m, p = case
    prob = S.make_problem(d, n, m, p, seed=9)
    ref = single_system(prob)
    w_ref = P.apply_schur(ref, prob["uhat"])
    eb = partition(d, n, prob["N"], world)
    plans = [rank_plan(prob["elem_face"], prob["face_elem"], prob["face_slot"], eb, r)
             for r in range(world)]
    systems = [RankSystem(prob, pl, device=0) for pl in plans]
    t = prob["t"]
    us = [torch.as_tensor(local_trace(prob["uhat"], pl, t), device="cuda") for pl in plans]
    ws = group_apply(systems, us)
    for pl, w in zip(plans, ws):
        assert np.array_equal(w.cpu().numpy(), local_trace(w_ref, pl, t))
    # and repeated applies are deterministic
    ws2 = group_apply(systems, us)
    assert all(torch.equal(a, b) for a, b in zip(ws, ws2))


def test_single_rank_plan_matches_plain_system(gpu):
    prob = S.make_problem(2, 8, 2, 2, seed=1)
    pl = rank_plan(prob["elem_face"], prob["face_elem"], prob["face_slot"],
                   np.array([0, prob["N"]]), 0)
    rs = RankSystem(prob, pl, device=0)
    ref = single_system(prob)
    u = torch.as_tensor(prob["uhat"], device="cuda")
    assert torch.equal(rs.apply(u), P.apply_schur(ref, u))
    assert np.array_equal(rs.f_dev.cpu().numpy(), ref.f_vec)


@pytest.mark.parametrize("split", [None, 0, 37, 64])
def test_single_rank_nccl_communicator(gpu, split, monkeypatch):
    """The NCCL path (dlopen, ncclCommInitRank, grouped halo calls, all-gathered
    batched reductions, GMRES with CGS2) on a one-rank communicator: bitwise the
    plain single-GPU apply, the solve within tolerance.  `split` forces the interior / halo macro
    split of the apply (macros [split, N) on the second stream, overlapping the
    halo exchange; [0, split) after it)."""
    if split is not None:
        monkeypatch.setenv("MEHDG_SPLIT_AT", str(split))
    # the multi-rank GMRES uses the grid-wide dot kernels, the plain system the
    # one-CTA MGS for a vector this short: the same partials in the same order
    prob = S.make_problem(2, 8, 2, 3, seed=4)
    pl = rank_plan(prob["elem_face"], prob["face_elem"], prob["face_slot"],
                   np.array([0, prob["N"]]), 0)
    rs = RankSystem(prob, pl, device=0, comm_id=nccl_unique_id())
    assert rs.has_comm
    ref = single_system(prob)
    u = torch.as_tensor(prob["uhat"], device="cuda")
    assert torch.equal(rs.apply(u), P.apply_schur(ref, u))
    assert np.array_equal(rs.f_dev.cpu().numpy(), ref.f_vec)
    # the multi-rank GMRES orthogonalises with CGS2 (two collectives per Arnoldi
    # step, krylov.cu) instead of the reference's MGS: same solve within tolerance
    x, info = rs.gmres(tol=1e-10)
    xr, ir = P.gmres(P.SchurOperator(ref), ref.f_device, P.SolverConfig(tol=1e-10),
                     precond=P.Preconditioner(ref))
    assert info["converged"] and abs(info["iterations"] - ir["iterations"]) <= 1
    xr = xr.cpu().numpy() if hasattr(xr, "cpu") else np.asarray(xr)
    xn = x.cpu().numpy()
    assert np.linalg.norm(xn - xr) <= 1e-9 * np.linalg.norm(xr)
