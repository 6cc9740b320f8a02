"""Form S_e and time / profile the matrix-based apply: python tools/mb_probe.py c2 [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_10917_b200 as P  # noqa: E402
from paper_2302_10917_b200 import synthetic as S  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
d, n, m, p = S.CONFIGS[name]
prob = S.make_problem(d, n, m, p, seed=0)
tables = {"nfe": d + 1, "elem_ufac": prob["elem_face"], "face_elem": prob["face_elem"],
          "face_slot": prob["face_slot"], "uidx": prob["uidx"], "F": prob["F"]}
sys_ = P.condense_arrays(prob["mesh"], prob["A"], None, prob["Be"], prob["R_u"], prob["D"],
                         prob["R_hat"], P.SolverConfig(tol=1e-10), tables=tables)
P.form_element_schur(sys_)
import torch  # noqa: E402
u = torch.from_numpy(prob["uhat"]).cuda()
for _ in range(3):
    w = P.apply_schur_mb(sys_, u)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(reps):
    w = P.apply_schur_mb(sys_, u)
torch.cuda.synchronize()
print(f"{name} mb apply ms={(time.perf_counter() - t0) / reps * 1e3:.4f}", flush=True)
