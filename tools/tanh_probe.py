"""Time the reference's top-level solve() on the tanh benchmark (device
assembly + condense + GMRES + reconstruct): python tools/tanh_probe.py [n] [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2302_10917_b200 as P  # noqa: E402
from paper_2302_10917_b200.assembly import StabilizationConfig, manufactured_tanh  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
problem = manufactured_tanh(0.4, (1.0, 1.0))
mesh = P.build_structured_macro_mesh(2, n, 2)
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sol, sys_ = P.solve(mesh, problem, StabilizationConfig(), P.SolverConfig(tol=1e-10), 3)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"solve n={n}: {dt:.3f} s, {sol.report.iterations} it, timings "
          f"{ {k: round(v, 4) for k, v in sys_.timings.items()} }", flush=True)
