"""Time the batched LU alone on one config: python tools/lu_probe.py c2 [reps].

MEHDG_LU=tile|cta selects the kernel (see csrc/lu.cu launch_lu).  Used
for kernel design points and as the ncu target for the LU."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_10917_b200 as P  # noqa: E402
from paper_2302_10917_b200 import synthetic as S  # noqa: E402
from paper_2302_10917_b200._lib import check, lib  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
d, n, m, p = S.CONFIGS[name]
prob = S.make_problem(d, n, m, p, seed=0)
tables = {"nfe": d + 1, "elem_ufac": prob["elem_face"], "face_elem": prob["face_elem"],
          "face_slot": prob["face_slot"], "uidx": prob["uidx"], "F": prob["F"]}
sys_ = P.condense_arrays(prob["mesh"], prob["A"], None, prob["Be"], prob["R_u"], prob["D"],
                         prob["R_hat"], P.SolverConfig(tol=1e-10), tables=tables)
N, Q = prob["N"], prob["Q"]


def run(tag):
    ts = []
    for i in range(reps):
        ms = C.c_float()
        check(lib.mh_refactorize_local(sys_.handle, C.byref(ms)), "lu")
        ts.append(ms.value)
    best = min(ts[1:] or ts)
    print(f"LU {name} Q={Q} N={N} {tag} ms={best:.3f} "
          f"TFLOP/s={2 / 3 * Q**3 * N / best / 1e9:.2f} all={np.round(ts, 3).tolist()}", flush=True)


run(f"variant={os.environ.get('MEHDG_LU', 'default')}")
# optional sweep of tuning environment variables, e.g.
#   python tools/lu_probe.py c2 4 MEHDG_LU_CTAS=1,2,3,4 MEHDG_LU_SCR=0,1
import itertools  # noqa: E402
knobs = [(a.split("=")[0], a.split("=")[1].split(",")) for a in sys.argv[3:]]
for combo in itertools.product(*[v for _, v in knobs]):
    for (k, _), v in zip(knobs, combo):
        os.environ[k] = v
    run(" ".join(f"{k}={v}" for (k, _), v in zip(knobs, combo)))
