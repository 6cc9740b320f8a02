import sys, time, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2302_10917_b200 as P
from paper_2302_10917_b200 import synthetic as S
prob = S.config_problem("c2")
sys_, cfg = None, None
tables = {"nfe": 3, "elem_ufac": prob["elem_face"], "face_elem": prob["face_elem"],
          "face_slot": prob["face_slot"], "uidx": prob["uidx"], "F": prob["F"]}
sys_ = P.condense_arrays(prob["mesh"], prob["A"], None, prob["Be"], prob["R_u"], prob["D"],
                         prob["R_hat"], P.SolverConfig(tol=1e-10), tables=tables)
n = sys_.zhat
up = torch.empty(n, dtype=torch.float64, pin_memory=True); up.copy_(torch.from_numpy(prob["uhat"]))
wp = torch.empty(n, dtype=torch.float64, pin_memory=True)
ud = torch.empty(n, dtype=torch.float64, device="cuda")
for name, fn in [("h2d", lambda: ud.copy_(up, non_blocking=True)), ("d2h", lambda: wp.copy_(ud, non_blocking=True))]:
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(50): fn()
    torch.cuda.synchronize(); print(name, (time.perf_counter() - t0) / 50 * 1e3, "ms", n * 8 / ((time.perf_counter() - t0) / 50) / 1e9, "GB/s")
def dev():
    P.apply_schur(sys_, ud, out=torch.empty_like(ud))
for k in (20, 100):
    P.apply_schur_many(sys_, up.numpy(), out=wp.numpy(), repeat=3)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    P.apply_schur_many(sys_, up.numpy(), out=wp.numpy(), repeat=k)
    print("many", k, (time.perf_counter() - t0) / k * 1e3, "ms/step")
w = torch.empty_like(ud)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(100): P.apply_schur(sys_, ud, out=w)
torch.cuda.synchronize(); print("device only", (time.perf_counter() - t0) / 100 * 1e3)
print("stream", torch.cuda.current_stream())
