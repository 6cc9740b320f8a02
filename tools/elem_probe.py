"""Time the matrix-free apply alone: python tools/elem_probe.py c3 [reps] [KNOB=v1,v2 ...].

Knobs are environment variables read when a system is created (MEHDG_ELEM_CTAS, ...).
Prints applies/s and the element kernel's algorithmic GB/s per setting."""
import itertools
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_10917_b200 as P  # noqa: E402
from paper_2302_10917_b200 import synthetic as S  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
d, n, m, p = S.CONFIGS[name]
prob = S.make_problem(d, n, m, p, seed=0)
tables = {"nfe": d + 1, "elem_ufac": prob["elem_face"], "face_elem": prob["face_elem"],
          "face_slot": prob["face_slot"], "uidx": prob["uidx"], "F": prob["F"]}
sys_ = P.condense_arrays(prob["mesh"], prob["A"], None, prob["Be"], prob["R_u"], prob["D"],
                         prob["R_hat"], P.SolverConfig(tol=1e-10), tables=tables)
u = torch.as_tensor(prob["uhat"], device="cuda")
w = torch.empty_like(u)
N, Q, nc = prob["N"], prob["Q"], prob["nc"]
elem_bytes = N * (8 * Q * Q + 4 * Q + 8 * nc * Q + 16 * nc + 4 * (d + 1))
st = torch.cuda.current_stream()


def run(tag):
    for _ in range(3):
        P.apply_schur(sys_, u, out=w)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(reps):
        P.apply_schur(sys_, u, out=w)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{name} {tag}: {1e3 / ms:.1f} applies/s, {ms:.3f} ms, "
          f"element-bytes rate {elem_bytes / ms / 1e6:.0f} GB/s, |w|={float(w.norm()):.12e}",
          flush=True)


run("default")
knobs = [(a.split("=")[0], a.split("=")[1].split(",")) for a in sys.argv[3:]]
for combo in itertools.product(*[v for _, v in knobs]):
    for (k, _), v in zip(knobs, combo):
        os.environ[k] = v
    run(" ".join(f"{k}={v}" for (k, _), v in zip(knobs, combo)))
