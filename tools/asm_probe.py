"""Time the device HDG assembly kernels: python tools/asm_probe.py [n] [m] [p] [reps]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_10917_b200 as P  # noqa: E402
from paper_2302_10917_b200.assembly import (StabilizationConfig, assemble_system_device,  # noqa: E402
                                            manufactured_tanh)

n, m, p = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (128, 2, 3)))
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
mesh = P.build_structured_macro_mesh(2, n, m)
prob = manufactured_tanh(0.4, (1.0, 1.0))
for supg in (False, True):
    ks = []
    for _ in range(reps):
        tm = {}
        blk = assemble_system_device(mesh, prob, StabilizationConfig(supg=supg), p, timings=tm)
        ks.append(tm["kernel_ms"])
        del blk
    nb = 8 * (mesh.n_elem * (blk_n := 3 * (m * p + 1) * (m * p + 2) // 2) ** 2)
    print(f"assembly n={n} m={m} p={p} supg={supg}: N={mesh.n_elem} kernel ms={min(ks):.3f} "
          f"host s={tm['host_s']:.3f} A bytes {nb / 1e9:.2f} GB -> {nb / min(ks) / 1e6:.0f} GB/s")
