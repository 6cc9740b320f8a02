"""GMRES(100) + D^-1 solve timing on one config; under ncu with
--profile-from-start off only the second (timed) solve is captured:

    python tools/gmres_probe.py c3
    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv python tools/gmres_probe.py c3
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2302_10917_b200 as P  # noqa: E402
from paper_2302_10917_b200 import synthetic as S  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
d, n, m, p = S.CONFIGS[name]
prob = S.make_problem(d, n, m, p, seed=0)
tables = {"nfe": d + 1, "elem_ufac": prob["elem_face"], "face_elem": prob["face_elem"],
          "face_slot": prob["face_slot"], "uidx": prob["uidx"], "F": prob["F"]}
cfg = P.SolverConfig(tol=1e-10)
sys_ = P.condense_arrays(prob["mesh"], prob["A"], None, prob["Be"], prob["R_u"], prob["D"],
                         prob["R_hat"], cfg, tables=tables)


def solve():
    return P.gmres(P.SchurOperator(sys_), sys_.f_device, cfg, precond=P.Preconditioner(sys_))


solve()
torch.cuda.synchronize()
ts = []
for r in range(3):
    if r == 2:
        torch.cuda.profiler.start()
    t0 = time.perf_counter()
    x, info = solve()
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
    if r == 2:
        torch.cuda.profiler.stop()
it = info["iterations"]
print(f"GMRES {name}: {it} iterations, {min(ts) * 1e3:.3f} ms ({min(ts) * 1e3 / it:.3f} ms/it), "
      f"all {[round(t * 1e3, 3) for t in ts]}")
