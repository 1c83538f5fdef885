"""run_gpu_batch at configs[2] (512^3 x 200) with two TBLOCK-in-place contexts
(40 arrays + gap each) vs one ping-pong TBLOCK context at a time: does the
stream overlap PCIe with the sweeps when ping-pong state fits only once?"""
import os
import sys
import time
from dataclasses import asdict

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1510_05218_b200 as P  # noqa: E402

d = P.GridDims(*[int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "512,512,512").split(",")])
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
n = int(sys.argv[3]) if len(sys.argv) > 3 else 4
import torch  # noqa: E402
print("mem_get_info", torch.cuda.mem_get_info(0), flush=True)
t = time.perf_counter()
host = P.generate_problem(d, P.GEN_RANDOM, 1)
out = [np.zeros_like(a) for a in host.fields]
print("generate", round(time.perf_counter() - t, 1), flush=True)
L = P.lib()
for a in host.arrays + out:
    L.thiim_gpu_pin_host(a.ctypes.data, a.nbytes)
for eng, depth in [(P.ENGINE_TBLOCK_INPLACE, 2), (P.ENGINE_AUTO, 3)]:
    o = P.GpuOptions(engine=eng)
    P.run_gpu_batch([host] * 2, iters, o, outputs=[out] * 2, depth=depth)  # warm-up
    t = time.perf_counter()
    r = P.run_gpu_batch([host] * n, iters, o, outputs=[out] * n, depth=depth)
    w = time.perf_counter() - t
    print(P.ENGINE_NAMES.get(eng), depth, n, "wall", round(w, 3), "e2e_mlups",
          round(d.interior_cells() * iters * n / w / 1e6, 1),
          {k: (round(v, 4) if isinstance(v, float) else v) for k, v in asdict(r).items()},
          flush=True)
