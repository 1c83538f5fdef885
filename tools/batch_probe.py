"""Times run_gpu_batch on the configs[1] problem for several depths / batch
sizes and prints each BatchReport (diagnostics for the e2e pipeline)."""
import os
import sys
import time
from dataclasses import asdict

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1510_05218_b200 as P  # noqa: E402

d = P.GridDims(*[int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "256,256,256").split(",")])
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
host = P.generate_problem(d, P.GEN_RANDOM, 1)
out = [np.zeros_like(a) for a in host.fields]
L = P.lib()
t = time.perf_counter()
for a in host.arrays + out:
    L.thiim_gpu_pin_host(a.ctypes.data, a.nbytes)
print("pin", round(time.perf_counter() - t, 3), flush=True)
for depth, n in [(3, 2), (3, 5), (3, 5), (2, 5), (1, 5), (3, 10)]:
    t = time.perf_counter()
    r = P.run_gpu_batch([host] * n, iters, outputs=[out] * n, depth=depth)
    w = time.perf_counter() - t
    print(depth, n, "wall", round(w, 3), {k: (round(v, 4) if isinstance(v, float) else v)
                                           for k, v in asdict(r).items()}, flush=True)
