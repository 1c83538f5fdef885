"""Two TBLOCK passes per grid shape, for ncu DRAM-traffic comparisons:

    ncu --kernel-name regex:k_tblock --metrics dram__bytes_read.sum,dram__bytes_write.sum,\
gpu__time_duration.sum --csv python tools/traffic_probe.py 256x256x256 252x176x256:z_chunk=256

Prints, per shape, the grid and the algorithmic bytes of one pass (832 B per
interior cell: 40 arrays read + 12 written, two steps)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1510_05218_b200 as P  # noqa: E402

for arg in sys.argv[1:]:
    kw = {}
    if ":" in arg:
        arg, o = arg.split(":", 1)
        kw = {k: int(v) for k, v in (x.split("=") for x in o.split(","))}
    nx, ny, nz = (int(v) for v in arg.split("x"))
    with P.GpuEngine(P.GridDims(nx, ny, nz), P.GpuOptions(engine=P.ENGINE_TBLOCK, **kw)) as e:
        e.generate(P.GEN_RANDOM, 1)
        st = e.step(2)
        st = e.step(2)
    print(json.dumps({"grid": [nx, ny, nz], "opts": kw, "algorithmic_bytes": 832 * nx * ny * nz,
                      "mlups": round(st.mlups, 1)}), flush=True)
