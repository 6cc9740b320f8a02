"""bench.py --impl reference: the UNMODIFIED reference solver on the host cores.

The reference (`mehdg`, pure Python + numpy/scipy) is installed once, offline,
into ``baseline/_ref`` (``python -m pip install --no-index --no-build-isolation
--no-deps --target baseline/_ref <copy of /root/reference/pkg>``; bench's
``__graft_entry__.build()`` does it when the directory is missing and the
reference is present).  ``baseline/_ref`` is git-ignored but travels to the GPU
box with the repo snapshot.

What runs, per BASELINE.md section 3 / SURVEY.md 8(d):
  * the mesh: ``mehdg.mesh.build_structured_macro_mesh(2, n, m)`` for d = 2; the
    reference has no 3-D skeleton (mesh.py:372-375), so for d = 3 the solver is
    handed the oracle's skeleton restatement duck-typed (``oracle/mesh_oracle``);
  * the blocks: the seeded BASELINE generator (``synthetic_gen.py``, pure numpy,
    loaded by file path so the product package and its CUDA library are never
    imported), injected through ``mehdg.assembly.LocalOperators`` /
    ``FaceOperator`` exactly as SURVEY 8(c) describes (op.B = B_e^T, op.C = B_e);
  * ``mehdg.schur_solver.condense`` (getrf of every block + reduced RHS), then
    W + K timed ``mehdg.schur_solver.apply_schur`` calls with ``workers=1`` and
    again with ``workers=os.cpu_count()`` (the reference's own WorkerPool,
    schur_solver.py:59-102); the line's value is the faster of the two.

Nothing here imports ``paper_2302_10917_b200``; the line records
``product_loaded`` from ``sys.modules`` and ``/proc/self/maps``.
"""

from __future__ import annotations

import importlib.util
import json
import os
import platform
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"


def _load_gen():
    path = ROOT / "paper_2302_10917_b200" / "synthetic_gen.py"
    spec = importlib.util.spec_from_file_location("mehdg_bench_synthetic_gen", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


class _Side:
    __slots__ = ("macro",)

    def __init__(self, macro):
        self.macro = macro


class _Face:
    """Duck-typed ``SkeletonFace``: the solver reads id, tag and sides() only
    (schur_solver.py:198-241)."""

    __slots__ = ("id", "tag", "_sides")

    def __init__(self, fid, tag, sides):
        self.id, self.tag, self._sides = fid, tag, sides

    def sides(self):
        return self._sides


class _Macro:
    __slots__ = ("m",)

    def __init__(self, m):
        self.m = m


class _Mesh:
    def __init__(self, skeleton, n_macros, m):
        self.skeleton = skeleton
        self.macro_elements = [_Macro(m) for _ in range(n_macros)]


def reference_mesh(d, n, m, n_macros=None):
    """(mesh for the solver, per-macro face ids in local-face order, N).

    ``n_macros``: restrict to the slab of macros [0, n_macros) (faces whose
    left side lies in it; right sides beyond it dropped) -- used only when the
    whole workload does not fit the host or the time budget."""
    from mehdg import mesh as RM

    if d == 2:
        M = RM.build_structured_macro_mesh(2, n, m)
        N = len(M.macro_elements)
        elem_faces = [[M.macro_elements[e].faces[k][0] for k in range(3)] for e in range(N)]
        faces = [(f.id, f.tag, [s.macro for s in f.sides()]) for f in M.skeleton]
        if n_macros is None:
            return M, elem_faces, N
    else:
        sys.path.insert(0, str(ROOT))
        from oracle.mesh_oracle import structured_skeleton

        sk = structured_skeleton(3, n)
        N = sk["elem_verts"].shape[0]
        elem_faces = sk["elem_face"].tolist()
        tags = {0: "interior", 1: "D", 2: "N"}
        faces = []
        for fid in range(sk["face_tag"].shape[0]):
            s = [int(sk["face_left"][fid, 0])]
            if sk["face_right"][fid, 0] >= 0:
                s.append(int(sk["face_right"][fid, 0]))
            faces.append((fid, tags[int(sk["face_tag"][fid])], s))
    e1 = N if n_macros is None else min(N, n_macros)
    skel = [_Face(fid, tag, [_Side(e) for e in s if e < e1])
            for fid, tag, s in faces if s[0] < e1]
    return _Mesh(skel, e1, m), elem_faces[:e1], e1


def inject(gen, mesh, elem_faces, N_full, Q, t, nc, seed):
    """LocalOperators / FaceOperator of the reference from the
    seeded generator; unknown faces numbered in skeleton order (the D blocks
    are drawn by that index, as the GPU path does)."""
    from mehdg import assembly as RA

    N = len(elem_faces)
    A, Be, Ru = gen.gen_macros(N_full, Q, nc, seed, 0, N)
    uidx, F = {}, 0
    for f in mesh.skeleton:
        if f.tag != "D":
            uidx[f.id] = F
            F += 1
    # D blocks are drawn by unknown-face index (the GPU path's numbering on the
    # whole mesh); a slab sample (c4 / c5, timing only) takes the first F draws
    D = gen.gen_faces(F, t, seed)
    local_ops = []
    for e in range(N):
        slots = [(fid, slice(k * t, (k + 1) * t)) for k, fid in enumerate(elem_faces[e])]
        local_ops.append(RA.LocalOperators(
            macro_id=e, A=A[e], B=np.ascontiguousarray(Be[e].T), C=Be[e], R_u=Ru[e],
            face_slots=slots, storage="dense"))
    face_ops = {fid: RA.FaceOperator(face_id=fid, D=D[u], R_hat=np.zeros(t), tag="interior")
                for fid, u in uidx.items()}
    return local_ops, face_ops, F


def host_info(workers):
    info = {"cpu_count": os.cpu_count(), "workers_timed": workers,
            "python": platform.python_version(), "numpy": np.__version__}
    try:
        import scipy

        info["scipy"] = scipy.__version__
    except ImportError:
        pass
    try:
        from threadpoolctl import threadpool_info

        info["blas"] = [{k: d.get(k) for k in ("internal_api", "version", "num_threads",
                                               "threading_layer", "architecture")}
                        for d in threadpool_info()]
    except ImportError:
        pass
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return info


def product_loaded() -> bool:
    if any(k.startswith("paper_2302_10917_b200") for k in sys.modules):
        return True
    try:
        return "libmehdg_b200" in Path("/proc/self/maps").read_text()
    except OSError:
        return False


def run(config, d, n, m, p, seed, steps, warmup, budget_s=150.0, emit=print, workers=None):
    if not (REF / "mehdg").is_dir():
        emit(json.dumps({"impl": "reference",
                         "unavailable": "baseline/_ref/mehdg missing (install the reference: "
                                        "python -c 'import __graft_entry__ as g; g.build()')"}))
        return 0
    sys.path.insert(0, str(REF))
    from mehdg import schur_solver as R

    gen = _load_gen()
    Q, t, nc = gen.block_sizes(d, m, p)
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    # c4 / c5 need 130-350+ GB of host RAM in the reference layout (BASELINE.md
    # section 3): time a slab of about 16k macros and extrapolate per macro
    N_full = {2: 2 * n * n, 3: 6 * n ** 3}[d]
    slab = None if N_full * (3 * Q * Q + 2 * nc * Q) * 8 < 24e9 else 16384
    mesh, elem_faces, N = reference_mesh(d, n, m, slab)
    t_mesh = time.perf_counter() - t0
    t0 = time.perf_counter()
    local_ops, face_ops, F = inject(gen, mesh, elem_faces, N_full, Q, t, nc, seed)
    t_inject = time.perf_counter() - t0
    cfg = R.SolverConfig(tol=1e-10, workers=1)
    t0 = time.perf_counter()
    sys_ = R.condense(mesh, local_ops, face_ops, cfg)
    t_condense = time.perf_counter() - t0
    uhat = np.random.default_rng([seed, 2]).standard_normal(sys_.zhat)

    # each setting's first warm-up apply is its cost estimate; each timed
    # setting gets `budget_s` seconds (the GIL-bound multi-worker one, ~3x
    # slower than workers=1 at c2, half of it), so the arm ends within a few
    # minutes -- at the driver's --steps 20 --warmup 5 on c2 (~1.4-1.8 s per
    # apply) workers=1 runs all W + K applies
    scale = N_full / N
    results = {}
    for workers in (sorted({1, cores}) if workers is None else [workers]):
        sys_.pool = R.WorkerPool(workers)
        bud = budget_s if workers == 1 else budget_s / 2
        t0 = time.perf_counter()
        R.apply_schur(sys_, uhat)
        t_first = time.perf_counter() - t0
        k_steps = steps
        if (steps + warmup - 1) * t_first > bud:  # keep the arm bounded
            k_steps = max(1, int(bud / t_first))
        for _ in range(warmup - 1 if k_steps == steps else 0):
            R.apply_schur(sys_, uhat)
        times = []
        for _ in range(k_steps):
            t0 = time.perf_counter()
            R.apply_schur(sys_, uhat)
            times.append(time.perf_counter() - t0)
        sys_.pool.close()
        results[workers] = {"apply_s_mean": float(np.mean(times)), "steps_timed": k_steps,
                            "applies_per_s": 1.0 / (float(np.mean(times)) * scale)}
    best_w = max(results, key=lambda w: results[w]["applies_per_s"])
    value = results[best_w]["applies_per_s"]
    ms = 1e3 / value
    lu_gflops = (2.0 / 3.0) * Q ** 3 * N / t_condense / 1e9  # condense = getrf + RHS
    sample = (f"unmodified mehdg.schur_solver (baseline/_ref) condense + apply_schur on "
              f"{'the whole workload' if slab is None else f'macros [0,{N}) of {N_full} (x{scale:.2f}, extrapolated per macro)'}"
              f" ({N} macros, {F} unknown faces, zhat {sys_.zhat}); workers "
              + ", ".join(f"{w}: {r['applies_per_s']:.3f} applies/s over {r['steps_timed']} steps"
                          for w, r in sorted(results.items())))
    line = {"impl": "reference",
            "metric": "Schur-operator applies/sec & HBM GB/s (% roofline); batched LU GFLOP/s fp64",
            "value": value, "unit": "applies/s", "n_gpus": 1, "steps": steps,
            "warmup": warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE generator, numpy PCG64)",
            "config": {"workload": f"BASELINE {config}: d={d} n={n} m={m} p={p} fp64 seed={seed}",
                       "N_macros": N_full, "Q": Q, "t": t, "nc": nc,
                       "operator": "reference apply_schur (D - C A^-1 B, per-macro lu_solve)",
                       "parallelism": f"host, WorkerPool workers={best_w}"},
            "cpu_baseline": {"value": value, "unit": "applies/s", "cores": best_w,
                             "kind": "reference", "sample": sample,
                             "by_workers": {str(w): r for w, r in results.items()},
                             "condense_s": t_condense, "lu_gflops_condense": lu_gflops,
                             "setup_s": {"mesh": t_mesh, "inject": t_inject},
                             "extrapolated": slab is not None},
            "e2e": {"value": value, "unit": "applies/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "host": host_info(sorted(results)),
            "product_loaded": product_loaded()}
    if line["product_loaded"]:
        raise RuntimeError("reference arm loaded the product package")
    emit(json.dumps(line))
    return 0


if __name__ == "__main__":
    # python baseline/reference_arm.py CONFIG [--steps K] [--warmup W] [--workers N]
    # (bench.py's cpu_baseline leg runs it in a separate process: the reference
    # alone, workers=1, the whole workload)
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--workers", type=int, default=None)
    ap.add_argument("--budget", type=float, default=60.0)
    a = ap.parse_args()
    d, n, m, p = _load_gen().CONFIGS[a.config]
    sys.exit(run(a.config, d, n, m, p, a.seed, a.steps, a.warmup, budget_s=a.budget,
                 workers=a.workers))
