import cProfile, pstats, time, sys
sys.path.insert(0, '.')
import paper_2302_10917_b200 as P
from paper_2302_10917_b200 import synthetic as S
import torch
prob = S.make_problem(2, 128, 4, 3, seed=0)
tables = {"nfe": 3, "elem_ufac": prob["elem_face"], "face_elem": prob["face_elem"],
          "face_slot": prob["face_slot"], "uidx": prob["uidx"], "F": prob["F"]}
cfg = P.SolverConfig(tol=1e-10)
torch.zeros(1, device="cuda")
t0 = time.perf_counter()
P.condense_arrays(prob["mesh"], prob["A"], None, prob["Be"], prob["R_u"], prob["D"], prob["R_hat"], cfg, tables=tables)
torch.cuda.synchronize()
print("first condense s", time.perf_counter() - t0)
pr = cProfile.Profile(); pr.enable()
t0 = time.perf_counter()
sys_ = P.condense_arrays(prob["mesh"], prob["A"], None, prob["Be"], prob["R_u"], prob["D"], prob["R_hat"], cfg, tables=tables)
torch.cuda.synchronize()
print("condense s", time.perf_counter() - t0)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
