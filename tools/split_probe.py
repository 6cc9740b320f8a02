"""Time the apply with the split element kernel: python tools/split_probe.py c5n20 [reps]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_10917_b200 as P  # noqa: E402
from paper_2302_10917_b200 import synthetic as S  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
d, n, m, p = S.CONFIGS[name]
prob = S.make_problem(d, n, m, p, seed=0)
tables = {"nfe": d + 1, "elem_ufac": prob["elem_face"], "face_elem": prob["face_elem"],
          "face_slot": prob["face_slot"], "uidx": prob["uidx"], "F": prob["F"]}
sys_ = P.condense_arrays(prob["mesh"], prob["A"], None, prob["Be"], prob["R_u"], prob["D"],
                         prob["R_hat"], P.SolverConfig(tol=1e-10), tables=tables)
import torch  # noqa: E402
u = torch.from_numpy(prob["uhat"]).cuda()
w = torch.empty_like(u)
for _ in range(5):
    P.apply_schur(sys_, u, out=w)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(reps):
    P.apply_schur(sys_, u, out=w)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / reps
print(f"{name} split={os.environ.get('MEHDG_ELEM_SPLIT', '0')} ctas={os.environ.get('MEHDG_ELEM_SPLIT_CTAS', '-')} "
      f"ms/apply={dt * 1e3:.3f}", flush=True)
