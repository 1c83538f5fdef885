"""Race stress for the TMA ring's slot release (thiim_ring.cuh): many random
shapes / seeds / step counts through the fused, TBLOCK (depth 2 and 3), TBLOCK-in-place (random
sub-range lengths), table and multi-slab (peer-store) engines,
each compared bitwise with the C oracle.  Prints one JSON line with the
number of cases and failures.  Test infrastructure: imports oracle/.

    python tools/stress_ring.py --seconds 120
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1510_05218_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=120)
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--only", default="", help="comma list of fused,tblock,inplace,tblock3,table,table-fused,slabs,slabs-table")
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    t_end = time.time() + a.seconds
    cases = fails = 0
    bad = []
    while time.time() < t_end:
        d = P.GridDims(int(rng.integers(4, 120)), int(rng.integers(4, 90)), int(rng.integers(4, 70)))
        steps = int(rng.integers(1, 6))
        seed = int(rng.integers(1, 1 << 30))
        layered = bool(rng.integers(0, 2)) or a.only in ("table", "table-fused")
        kind = P.GEN_LAYERED if layered else P.GEN_RANDOM
        ref = P.generate_problem(d, kind, seed)
        O.c_step((d.nx, d.ny, d.nz), ref.arrays, steps, threads=8)
        runs = [("fused", P.GpuOptions(engine=P.ENGINE_FUSED)),
                ("tblock", P.GpuOptions(engine=P.ENGINE_TBLOCK)),
                ("inplace", P.GpuOptions(engine=P.ENGINE_TBLOCK_INPLACE)),
                ("tblock3", P.GpuOptions(engine=P.ENGINE_TBLOCK, time_block=3))]
        ip_L = int(rng.integers(2, max(3, d.nz + 1)))  # sub-range length of the in-place run
        if layered:
            runs.append(("table", P.GpuOptions(coeff_layout=P.COEFF_TABLE, n_materials=6,
                                               engine=P.ENGINE_TBLOCK)))
            runs.append(("table-fused", P.GpuOptions(coeff_layout=P.COEFF_TABLE, n_materials=6,
                                                     engine=P.ENGINE_FUSED)))
        # z-slabs of one context on this device: peer stores into the neighbours'
        # halos from the TBLOCK kernel, passes ordered by stream events
        ns = int(rng.integers(2, 4))
        if d.nz >= 4 * ns:
            runs.append(("slabs", P.GpuOptions(engine=P.ENGINE_TBLOCK, n_gpus=ns, same_device=1)))
            if layered:
                runs.append(("slabs-table", P.GpuOptions(engine=P.ENGINE_TBLOCK, n_gpus=ns,
                                                         same_device=1, coeff_layout=P.COEFF_TABLE,
                                                         n_materials=6)))
        if a.only:
            runs = [r for r in runs if r[0] in a.only.split(",")]
        for name, o in runs:
            out = P.generate_problem(d, kind, seed)
            if name == "inplace":
                os.environ["THIIM_INPLACE_TB"] = str(ip_L)
            else:
                os.environ.pop("THIIM_INPLACE_TB", None)
            with P.GpuEngine(d, o) as e:
                e.generate(kind, seed)
                e.step(steps)
                e.download_fields(out)
            cases += 1
            diff = P.compare_states(ref, out)
            if not diff.bitwise_equal:
                fails += 1
                bad.append([name, d.nx, d.ny, d.nz, steps, seed, layered])
    print(json.dumps({"stress": "ring release", "cases": cases, "failures": fails, "bad": bad[:20]}))
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
