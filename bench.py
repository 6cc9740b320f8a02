"""Benchmark of the B200 Schur-operator path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

One *step* is one matrix-free Schur-operator apply w = (D - C A^-1 B) uhat over
every macro and unknown face of the workload (BASELINE configs[1] = c2 on one
GPU: d=2, n=128, m=4, p=3, N=32768 macros, Q=91, t=13, zhat=635,648), with the
seeded synthetic blocks of paper_2302_10917_b200.synthetic resident in HBM.
The blocks (3.2 GB per apply) are far larger than the 126 MB L2, so no L2
flush is needed between steps.

Prints ONE JSON line (rank 0):  value = applies/s of the whole job (device
time, CUDA events on the library's stream, max over ranks), plus
  roofline      the element kernel (dominant) vs the measured HBM copy peak
  e2e           the same metric through the public API with pinned host buffers
                (H2D of uhat and D2H of w inside every step)
  lu            batched LU GFLOP/s (fp64) of the factorisation kernel
  solve         GMRES(100) + D^-1 to 1e-10: iterations and seconds
  cpu_baseline  the reference's own CPU path (the unmodified solver from
                baseline/_ref, one core, separate process) on the whole
                workload on this host; the oracle port when it is not installed.
`--impl reference` times the UNMODIFIED reference (`mehdg`, installed offline
into baseline/_ref) on the host cores: condense + apply_schur at workers=1 and
workers=cpu_count (baseline/reference_arm.py; never imports this package).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
# stdout carries the one JSON line: NCCL's version banner (the image sets
# NCCL_DEBUG=VERSION, which prints to stdout) is turned off, other NCCL log
# lines go to stderr
if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
    os.environ["NCCL_DEBUG"] = "WARN"
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")

BASELINE_METRIC = "Schur-operator applies/sec & HBM GB/s (% roofline); batched LU GFLOP/s fp64"
UNIT = "applies/s"


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def fp64_peak_tflops() -> tuple:
    """The measured fp64 DMMA peak (tools/fp64_peak.cu, profiles/r1_fp64_peak.txt)."""
    p = ROOT / "profiles" / "r1_fp64_peak.txt"
    best = 0.0
    if p.exists():
        for line in p.read_text().splitlines():
            if line.startswith("DMMA") and "TFLOP/s" in line:
                try:
                    best = max(best, float(line.split(":")[1].split()[0]))
                except (IndexError, ValueError):
                    pass
    if best > 0:
        return best, "measured DMMA.8x8x4 issue-bound peak (profiles/r1_fp64_peak.txt)"
    return 37.0, "fallback (HGX B200 fp64 tensor figure / 8)"


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None
        self.active = False
        self._thr = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self._thr = threading.Thread(target=self._read, daemon=True)
        self._thr.start()

    def _read(self):
        for line in self.proc.stdout:
            if self.active:
                self.samples.append(line.strip())

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for s in self.samples:
            parts = [x.strip() for x in s.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# distributed plumbing

def dist_setup(slabs: bool = False):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or slabs:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# CPU oracle leg (bounded sample of the same workload)

def oracle_sample(prob: dict, n_macros: int, threads: int = 1, first: int = 0):
    """An OracleSystem over macros [first, first + n_macros) of the workload and the
    unknown faces whose left side lies in it (right sides outside are dropped)."""
    from oracle import solver_oracle as SO

    e0 = min(first, prob["N"])
    e1 = min(first + n_macros, prob["N"])
    ns = e1 - e0
    fe, fs = prob["face_elem"], prob["face_slot"]
    keep = (fe[:, 0] >= e0) & (fe[:, 0] < e1)
    fidx = np.nonzero(keep)[0]
    remap = -np.ones(prob["F"], np.int64)
    remap[fidx] = np.arange(fidx.size)
    ef = prob["elem_face"][e0:e1].astype(np.int64)
    ef = np.where(ef >= 0, remap[np.maximum(ef, 0)], -1)
    fe_s = fe[fidx].astype(np.int64).copy() - e0
    fs_s = fs[fidx].astype(np.int64).copy()
    outside = (fe_s[:, 1] < 0) | (fe_s[:, 1] >= ns) | (fe[fidx, 1] < 0)
    fe_s[outside, 1] = -1
    fs_s[outside, 1] = -1
    o = SO.OracleSystem(prob["A"][e0:e1], prob["B"][e0:e1], prob["C"][e0:e1], prob["R_u"][e0:e1],
                        prob["D"][fidx], prob["R_hat"][fidx], ef, fe_s, fs_s, prob["t"])
    return o, ns, int(fidx.size)


def cpu_baseline_leg(args, prob: dict) -> dict:
    """The reference's own CPU path on this host: the unmodified `mehdg` solver
    (baseline/_ref) in a separate process, workers=1, condense + `cpu_reps`
    timed applies of the WHOLE workload (~15 s at c2).  Without the installed
    reference: the oracle port, also on the whole workload."""
    ref = ROOT / "baseline" / "_ref" / "mehdg"
    if ref.is_dir():
        cmd = [sys.executable, str(ROOT / "baseline" / "reference_arm.py"), args.config,
               "--steps", str(args.cpu_reps), "--warmup", "1", "--workers", "1",
               "--seed", str(args.seed), "--budget", "60"]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        rec = next((json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")), None)
        if r.returncode == 0 and rec and "value" in rec:
            cb = rec["cpu_baseline"]
            return {"value": rec["value"], "unit": UNIT, "cores": 1, "kind": "reference",
                    "sample": cb["sample"], "extrapolated": cb["extrapolated"],
                    "condense_s": cb["condense_s"], "lu_gflops": cb["lu_gflops_condense"],
                    "host": rec.get("host")}
    cb = time_oracle(prob, prob["N"], reps=args.cpu_reps, threads=1)
    return {"value": cb["applies_per_s"], "unit": UNIT, "cores": 1, "kind": "port",
            "sample": (f"oracle port (per-macro scipy LAPACK loop) on the whole workload "
                       f"({cb['sample_macros']} macros, {cb['sample_faces']} faces), mean of "
                       f"{cb['reps']} applies"),
            "extrapolated": cb["scale"] != 1.0, "lu_gflops": cb["lu_gflops"]}


def time_oracle(prob: dict, n_macros: int, reps: int, threads: int):
    """Oracle factorisation + `reps` applies on the sample; returns a dict."""
    from threadpoolctl import threadpool_limits

    with threadpool_limits(limits=threads):
        o, ns, fs = oracle_sample(prob, n_macros)
        t0 = time.perf_counter()
        o.factorize()
        t_fac = time.perf_counter() - t0
        u = np.random.default_rng(1).standard_normal(o.zhat)
        o.apply(u)
        times = []
        for _ in range(reps):
            t0 = time.perf_counter()
            o.apply(u)
            times.append(time.perf_counter() - t0)
    scale = prob["N"] / ns
    t_apply = float(np.mean(times)) * scale
    lu_gflops = (2.0 / 3.0) * prob["Q"] ** 3 * ns / t_fac / 1e9
    return {"apply_s_full": t_apply, "applies_per_s": 1.0 / t_apply, "sample_macros": ns,
            "sample_faces": fs, "scale": scale, "lu_gflops": lu_gflops, "reps": reps,
            "sample_apply_s": float(np.mean(times))}


# ---------------------------------------------------------------------------

def config_block(name, prob, world, slabs=False):
    return {"workload": f"BASELINE {name}: d={prob['d']} n={prob['n']} m={prob['m']} "
                        f"p={prob['p']} fp64 seed={prob['seed']}",
            "N_macros": prob["N"], "Q": prob["Q"], "t": prob["t"], "nc": prob["nc"],
            "F_unknown": prob["F"], "zhat": prob["zhat"],
            "operator": "matrix-free D - C A^-1 B (C = B^T synthetic, B_e streamed once)",
            "l2_flush": "none needed: 3.2 GB of blocks per apply >> 126 MB L2",
            "parallelism": f"slabs{world} (NCCL halo)" if (world > 1 or slabs) else "single"}


def run_reference(args, world, rank):
    """--impl reference: the unmodified reference solver (baseline/_ref) on the
    host cores, same config / metric (baseline/reference_arm.py).  Under
    torchrun only rank 0 runs it."""
    if rank != 0:
        return 0
    sys.path.insert(0, str(ROOT / "baseline"))
    import reference_arm

    d, n, m, p = reference_arm._load_gen().CONFIGS[args.config]
    return reference_arm.run(args.config, d, n, m, p, args.seed, args.steps, args.warmup,
                             budget_s=args.ref_budget)


def build_local(args, world, rank, dev):
    """This rank's system: the whole problem at N=1, its slab at N>1."""
    import numpy as np

    import paper_2302_10917_b200 as P
    from paper_2302_10917_b200 import synthetic as S

    d, n, m, p = S.CONFIGS[args.config]
    t0 = time.perf_counter()
    if world == 1 and not args.slabs:
        prob = S.make_problem(d, n, m, p, seed=args.seed)
        t_gen = time.perf_counter() - t0
        tables = {"nfe": d + 1, "elem_ufac": prob["elem_face"], "face_elem": prob["face_elem"],
                  "face_slot": prob["face_slot"], "uidx": prob["uidx"], "F": prob["F"]}
        cfg = P.SolverConfig(tol=1e-10, device=dev)
        t0 = time.perf_counter()
        sys_ = P.condense_arrays(prob["mesh"], prob["A"], None, prob["Be"], prob["R_u"],
                                 prob["D"], prob["R_hat"], cfg, tables=tables, device=dev)
        return prob, sys_, None, t_gen, time.perf_counter() - t0
    from paper_2302_10917_b200.distributed import RankSystem, broadcast_unique_id, local_trace
    from paper_2302_10917_b200.partition import partition, rank_plan

    prob = S.make_problem(d, n, m, p, seed=args.seed, with_blocks=False)
    eb = partition(d, n, prob["N"], world)
    plan = rank_plan(prob["elem_face"], prob["face_elem"], prob["face_slot"], eb, rank)
    A, Be, Ru = S.gen_macros(prob["N"], prob["Q"], prob["nc"], args.seed, plan.e0, plan.n_local)
    D = S.gen_faces_at(prob["F"], prob["t"], args.seed, plan.owned)  # owned faces only
    uh = S.gen_uhat(prob["zhat"], args.seed)
    prob["uhat_local"] = local_trace(uh, plan, prob["t"])
    t_gen = time.perf_counter() - t0
    cid = broadcast_unique_id(rank, dev)
    t0 = time.perf_counter()
    rs = RankSystem(prob, plan, device=dev, comm_id=cid,
                    blocks=dict(A=A, Be=Be, R_u=Ru, D=D, R_hat=np.zeros((plan.F_own, prob["t"]))))
    return prob, rs, plan, t_gen, time.perf_counter() - t0


def lu_block(lu_ms, lu_flops, N, Q, hbm_gbs):
    """Batched LU: GFLOP/s and the fraction of its roofline
    max(16 Q^2 N / BW, (2/3) Q^3 N / P_fp64)."""
    p64, p64_src = fp64_peak_tflops()
    lu_bytes = 16 * N * Q * Q  # A read once, L\U written once
    t_hbm = lu_bytes / (hbm_gbs * 1e9) * 1e3
    t_fp = lu_flops / (p64 * 1e12) * 1e3
    bound_ms = max(t_hbm, t_fp)
    return {"gflops": lu_flops / (lu_ms * 1e-3) / 1e9, "ms": lu_ms, "flops": lu_flops,
            "bytes": lu_bytes, "gbs": lu_bytes / (lu_ms * 1e-3) / 1e9,
            "roofline": {"bound": "hbm" if t_hbm >= t_fp else "fp64", "bound_ms": bound_ms,
                         "frac": bound_ms / lu_ms, "fp64_peak_tflops": p64,
                         "fp64_peak_source": p64_src, "hbm_peak_gbs": hbm_gbs}}


def run_ours(args, world, rank, local):
    import ctypes as C

    import torch

    import paper_2302_10917_b200 as P
    from paper_2302_10917_b200 import synthetic as S
    from paper_2302_10917_b200._lib import check, lib, ptr

    dev = local
    torch.cuda.set_device(dev)
    prob, sys_, plan, t_gen, t_condense = build_local(args, world, rank, dev)
    h = sys_.handle
    stream = torch.cuda.current_stream(dev)
    d = prob["d"]
    N, Q, nc, t, F = prob["N"], prob["Q"], prob["nc"], prob["t"], prob["F"]
    N_loc = N if plan is None else plan.n_local
    F_loc = F if plan is None else plan.F_own

    # ---- batched LU (this rank's blocks) ------------------------------------
    lu_ms = []
    for i in range(4):
        ms = C.c_float()
        check(lib.mh_refactorize_local(h, C.byref(ms)), "lu")
        if i:
            lu_ms.append(ms.value)
    lu_ms = max_over_ranks(float(sum(lu_ms) / len(lu_ms)), world)
    lu_flops = S.lu_flops(N, Q)

    # ---- device-resident applies --------------------------------------------
    u_host = prob["uhat"] if plan is None else prob["uhat_local"]
    u = torch.as_tensor(u_host, device=f"cuda:{dev}")
    w = torch.empty_like(u)
    sampler = ClockSampler(dev)
    sampler.start()
    # warm-up: at least W applies and at least 1 s of back-to-back applies right
    # before the timed region (clocks and power at their sustained state, no
    # idle gap), so a short timed window reports the sustained rate
    t_w = time.perf_counter()
    nw = 0
    while nw < args.warmup or time.perf_counter() - t_w < args.warmup_seconds:
        for _ in range(8):
            check(lib.mh_apply(h, ptr(u), ptr(w)), "apply")
        nw += 8
        torch.cuda.synchronize(dev)
    barrier(world)
    torch.cuda.synchronize(dev)
    check(lib.mh_profile_read(h, None, None, None, None), "profile")
    sampler.active = True
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    # per-kernel CUDA events (mh_profile) on every `pe`-th apply of the timed
    # region: the roofline's kernel durations, without an event pair around
    # every launch of every step
    pe = max(1, args.profile_every)
    sampled = 0
    e0.record(stream)
    for i in range(args.steps):
        if i % pe == 0:
            check(lib.mh_profile(h, 1), "profile")
            check(lib.mh_apply(h, ptr(u), ptr(w)), "apply")
            check(lib.mh_profile(h, 0), "profile")
            sampled += 1
        else:
            check(lib.mh_apply(h, ptr(u), ptr(w)), "apply")
    e1.record(stream)
    torch.cuda.synchronize(dev)
    sampler.active = False
    barrier(world)
    elapsed_ms = e0.elapsed_time(e1)
    el_ms, el_n, fa_ms, fa_n = C.c_double(), C.c_int64(), C.c_double(), C.c_int64()
    check(lib.mh_profile_read(h, C.byref(el_ms), C.byref(el_n), C.byref(fa_ms), C.byref(fa_n)),
          "profile")
    sampler.stop()
    elapsed_ms = max_over_ranks(elapsed_ms, world)
    ms_per_step = elapsed_ms / args.steps
    value = 1e3 / ms_per_step  # applies/s of the whole (global) operator

    bytes_apply = S.algorithmic_bytes_per_apply(N, Q, nc, d, F, t)
    elem_bytes = N_loc * (8 * Q * Q + 4 * Q + 8 * nc * Q + 16 * nc + 4 * (d + 1))
    elem_avg_ms = el_ms.value / max(el_n.value, 1)
    face_avg_ms = fa_ms.value / max(fa_n.value, 1)
    peaks = measured_peaks()
    achieved = elem_bytes / (elem_avg_ms * 1e-3) / 1e9
    traffic = None
    prof_json = ROOT / "profiles" / f"ncu_traffic_{args.config}.json"
    if prof_json.exists():
        try:
            traffic = json.loads(prof_json.read_text()).get("element_kernel_dram_bytes")
        except (ValueError, OSError):
            traffic = None

    # ---- end-to-end through the public API (pinned host buffers) -------------
    u_pin = torch.empty(u.numel(), dtype=torch.float64, pin_memory=True)
    u_pin.copy_(torch.from_numpy(u_host))
    w_pin = torch.empty(u.numel(), dtype=torch.float64, pin_memory=True)  # empty_like drops pinning
    e2e_steps = max(3, min(args.steps, 200))

    def e2e_step():
        if plan is None:  # numpy in -> numpy out; H2D + D2H inside the call
            return P.apply_schur(sys_, u_pin.numpy(), out=w_pin.numpy())
        ud = u_pin.to(f"cuda:{dev}", non_blocking=True)
        wd = sys_.apply(ud)
        w_pin.copy_(wd, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
        return w_pin

    for _ in range(2):
        e2e_step()
    barrier(world)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    e0.record(stream)
    for _ in range(e2e_steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    e2e_wall = time.perf_counter() - t0
    e2e_sync_ms = max_over_ranks(max(e0.elapsed_time(e1), e2e_wall * 1e3) / e2e_steps, world)

    # streaming form of the same public API: one call applies the operator to
    # e2e_steps host vectors; each step still copies its input in and its result
    # out (5 MB each way at c2), but the copies of steps i+1 / i-1 overlap the
    # apply of step i on the GPU's copy engines (mh_apply_host_many)
    def e2e_many(k):
        if plan is None:
            P.apply_schur_many(sys_, u_pin.numpy(), out=w_pin.numpy(), repeat=k)
        else:
            check(lib.mh_apply_host_many(h, k, ptr(u_pin), 0, ptr(w_pin), 0), "apply_many")

    e2e_many(3)
    barrier(world)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    e2e_many(e2e_steps)
    e2e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3 / e2e_steps, world)

    # ---- matrix-based mode (explicit element Schur blocks)
    mb = None
    if plan is None and not args.no_mb:
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        P.form_element_schur(sys_)
        torch.cuda.synchronize(dev)
        t_form = time.perf_counter() - t0
        e0.record(stream)  # the form kernel alone (S already allocated)
        P.form_element_schur(sys_)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        form_ms = e0.elapsed_time(e1)
        # two triangular solves with nc right-hand sides + the C Y product
        form_flops = N * (2.0 * Q * Q * nc + 2.0 * nc * nc * Q)
        for _ in range(3):
            check(lib.mh_apply_mb(h, ptr(u), ptr(w)), "apply_mb")
        mb_steps = max(10, args.steps // 2)
        e0.record(stream)
        for _ in range(mb_steps):
            check(lib.mh_apply_mb(h, ptr(u), ptr(w)), "apply_mb")
        e1.record(stream)
        torch.cuda.synchronize(dev)
        mb_ms = e0.elapsed_time(e1) / mb_steps
        mb_bytes = N * (8 * nc * nc + 16 * nc) + F * (8 * t * t + 32 * t)
        mb = {"applies_per_s": 1e3 / mb_ms, "ms_per_apply": mb_ms, "form_s": t_form,
              "form_kernel_ms": form_ms, "form_gflops": form_flops / form_ms / 1e6,
              "form_frac_fp64_peak": form_flops / (form_ms * 1e-3) / (fp64_peak_tflops()[0] * 1e12),
              "bytes_per_apply": mb_bytes, "gbs": mb_bytes / (mb_ms * 1e-3) / 1e9}

    # ---- full solve (GMRES + D^-1 to 1e-10); the first call allocates the
    # Krylov basis, the second is timed ----------------------------------------
    def run_solve():
        if plan is None:
            cfg = P.SolverConfig(tol=1e-10, device=dev)
            return P.gmres(P.SchurOperator(sys_), sys_.f_device, cfg,
                           precond=P.Preconditioner(sys_))
        return sys_.gmres(tol=1e-10)

    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    run_solve()
    torch.cuda.synchronize(dev)
    t_solve_first = time.perf_counter() - t0
    barrier(world)
    t0 = time.perf_counter()
    x, info = run_solve()
    torch.cuda.synchronize(dev)
    t_solve = max_over_ranks(time.perf_counter() - t0, world)

    # ---- device assembly of real HDG blocks: the tanh
    # manufactured case on a 2-D mesh, blocks assembled on the device, then the
    # reference's solve() driver end to end on a smaller mesh ------------------
    asm = None
    if plan is None and not args.no_asm:
        from paper_2302_10917_b200.assembly import (StabilizationConfig, assemble_system_device,
                                                    manufactured_tanh)
        problem = manufactured_tanh(0.4, (1.0, 1.0))
        n_a, m_a, p_a = 128, 2, 3
        mesh_a = P.build_structured_macro_mesh(2, n_a, m_a)
        assemble_system_device(mesh_a, problem, StabilizationConfig(), p_a, device=dev)  # warm
        tm = {}
        blk = assemble_system_device(mesh_a, problem, StabilizationConfig(), p_a, device=dev,
                                     timings=tm)
        N_a, nloc_a, t_a = mesh_a.n_elem, blk.nloc, blk.t
        F_a = int(blk.D.shape[0])
        out_bytes = 8 * (N_a * (nloc_a * nloc_a + 2 * nloc_a * 3 * t_a + nloc_a) + F_a * t_a * t_a)
        del blk
        torch.cuda.empty_cache()
        mesh_s = P.build_structured_macro_mesh(2, 32, m_a)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        sol, sys_s = P.solve(mesh_s, problem, StabilizationConfig(),
                             P.SolverConfig(tol=1e-10, device=dev), p_a)
        t_s = time.perf_counter() - t0
        asm = {"problem": "tanh (mehdg bench.py), kappa=0.4, a=(1,1), d=2 m=2 p=3",
               "assembly": {"n": n_a, "N_macros": N_a, "nloc": nloc_a, "nc": 3 * t_a,
                            "kernel_ms": tm["kernel_ms"], "host_s": tm["host_s"],
                            "macros_per_s": N_a / (tm["kernel_ms"] * 1e-3),
                            "bytes_written": out_bytes,
                            "gbs": out_bytes / (tm["kernel_ms"] * 1e-3) / 1e9},
               "solve": {"n": 32, "N_macros": mesh_s.n_elem, "zhat": sys_s.zhat,
                         "iterations": sol.report.iterations, "converged": sol.report.converged,
                         "seconds_total": t_s, "assemble_s": sys_s.timings.get("assemble")}}
        del sys_s, sol
        torch.cuda.empty_cache()

    line = {
        "metric": BASELINE_METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "warmup_detail": {"applies": nw, "min_seconds": args.warmup_seconds},
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE generator, numpy PCG64; blocks resident in HBM)",
        "config": config_block(args.config, prob, world, plan is not None),
        "hbm_gbs": bytes_apply / (ms_per_step * 1e-3) / 1e9,
        "hbm_frac": bytes_apply / (ms_per_step * 1e-3) / 1e9 / (peaks["hbm_gbs"] * world),
        "bytes_per_apply": bytes_apply,
        "roofline": {"bound": "hbm", "kernel": "element_kernel (gather+B^T+LU solve+C, per macro)",
                     "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                     "algorithmic_bytes_per_launch": elem_bytes, "avg_launch_ms": elem_avg_ms,
                     "face_kernel_avg_ms": face_avg_ms, "peak_source": peaks["source"]},
        "e2e": {"value": 1e3 / e2e_ms, "unit": UNIT, "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": prob["zhat"] * 8, "d2h_bytes_per_step": prob["zhat"] * 8,
                "api": "paper_2302_10917_b200.apply_schur_many(sys, uhat, out=w, repeat=steps) "
                       "(mh_apply_host_many) with pinned numpy buffers, host wall clock",
                "sync_value": 1e3 / e2e_sync_ms,
                "sync_api": "apply_schur(sys, uhat, out=w) per step (copies not overlapped)"
                if plan is None else "RankSystem.apply with pinned host copies per rank"},
        # element + face launches per apply (counted on the profiled applies) x steps
        "gpu_launches": int(round((el_n.value + fa_n.value) / max(sampled, 1) * args.steps)),
        "profiled_applies": sampled,
        "lu": lu_block(lu_ms, lu_flops, N, Q, peaks["hbm_gbs"]),
        "solve": {"iterations": info["iterations"], "converged": info["converged"],
                  "seconds": t_solve, "ms_per_iteration": t_solve * 1e3 / max(info["iterations"], 1),
                  "first_call_seconds": t_solve_first, "tol": 1e-10},
        "setup_s": {"generate": t_gen, "condense": t_condense},
        "mb_mode": mb,
        "hdg_assembly": asm,
        "clocks": sampler.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_leg(args, prob)
    if rank == 0:
        print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    # cpu_baseline leg of our arm: the reference on one core, condense + the
    # timed applies of the whole workload (~15 s at c2)
    ap.add_argument("--cpu-reps", type=int, default=3)
    ap.add_argument("--ref-budget", type=float, default=150.0,
                    help="--impl reference: seconds of timed applies per worker setting")
    ap.add_argument("--warmup-seconds", type=float, default=1.0,
                    help="minimum wall time of back-to-back warm-up applies")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-mb", action="store_true", help="skip the matrix-based mode timing")
    ap.add_argument("--profile-every", type=int, default=10,
                    help="per-kernel CUDA events on every k-th apply of the timed region")
    ap.add_argument("--slabs", action="store_true",
                    help="take the multi-rank path (RankSystem, NCCL communicator) even on "
                         "one rank; launch under torchrun")
    ap.add_argument("--no-asm", action="store_true",
                    help="skip the device HDG assembly / real-problem solve timing")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, local = (1, 0, 0)
    if args.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        return run_reference(args, world, rank)
    world, rank, local = dist_setup(args.slabs)
    try:
        return run_ours(args, world, rank, local)
    finally:
        if world > 1 or args.slabs:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
