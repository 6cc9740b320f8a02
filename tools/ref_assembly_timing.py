"""Time the reference's assemble_system (CPU, pure Python + numpy) on the
bench's assembly problem at a reduced size; run in the build container only
(it imports /root/reference):

    PYTHONPATH=/root/reference/pkg/src python tools/ref_assembly_timing.py [n]
"""
import sys
import time

from mehdg import assembly as RA
from mehdg import mesh as RM
from mehdg import schur_solver as R
from mehdg.bench import make_benchmark

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
case = make_benchmark("tanh", 0.4, (1.0, 1.0))
mesh = RM.build_structured_macro_mesh(2, n, 2)
pool = R.WorkerPool(1)
t0 = time.perf_counter()
lo, fo = R.assemble_system(mesh, case.problem(), RA.StabilizationConfig(), 3, pool)
t = time.perf_counter() - t0
print(f"reference assemble_system d=2 n={n} m=2 p=3: {len(lo)} macros + {len(fo)} faces in "
      f"{t:.2f} s = {len(lo) / t:.0f} macros/s (1 core)")
