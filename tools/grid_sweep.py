"""MLUP/s of the default engine over grid shapes (device time from the
library's CUDA events).  python tools/grid_sweep.py 256x256x256 252x253x256 ..."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1510_05218_b200 as P  # noqa: E402


def main():
    steps = int(os.environ.get("SWEEP_STEPS", "100"))
    for arg in sys.argv[1:]:
        opts = {}
        if ":" in arg:
            arg, o = arg.split(":", 1)
            opts = dict(kv.split("=") for kv in o.split(","))
        nx, ny, nz = (int(v) for v in arg.split("x"))
        d = P.GridDims(nx, ny, nz)
        kw = {k: int(v) for k, v in opts.items()}
        with P.GpuEngine(d, P.GpuOptions(**kw)) as e:
            e.generate(P.GEN_RANDOM, 1)
            e.step(steps)
            best = 0.0
            for _ in range(3):
                st = e.step(steps)
                best = max(best, st.mlups)
        print(json.dumps({"grid": [nx, ny, nz], "opts": kw, "mlups": round(best, 1),
                          "engine": st.engine}), flush=True)


if __name__ == "__main__":
    main()
