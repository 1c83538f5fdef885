"""Phase breakdown of one end-to-end run_gpu call on the c1 workload
(context create, upload from pinned host memory, 100 steps, download,
destroy).  Wall clock around each synchronous library call."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1510_05218_b200 as P  # noqa: E402


def main():
    d = P.GridDims(256, 256, 256)
    host = P.generate_problem(d, P.GEN_RANDOM, 1)
    t0 = time.perf_counter()
    for a in host.arrays:
        P.lib().thiim_gpu_pin_host(a.ctypes.data, a.nbytes)
    pin = time.perf_counter() - t0
    out = []
    for rep in range(3):
        t = [time.perf_counter()]
        e = P.GpuEngine(d, P.GpuOptions())
        t.append(time.perf_counter())
        e.upload(host)
        t.append(time.perf_counter())
        st = e.step(100)
        t.append(time.perf_counter())
        e.download_fields(host)
        t.append(time.perf_counter())
        e.close()
        t.append(time.perf_counter())
        ph = [round(1e3 * (b - a), 2) for a, b in zip(t, t[1:])]
        out.append(dict(zip(["create_ms", "upload_ms", "step_ms", "download_ms", "destroy_ms"], ph)))
    up_bytes = sum(a.nbytes for a in host.arrays)
    dn_bytes = sum(a.nbytes for a in host.arrays[:12])
    last = out[-1]
    print(json.dumps({"pin_ms": round(1e3 * pin, 1), "reps": out,
                      "upload_GBps": round(up_bytes / last["upload_ms"] / 1e6, 2),
                      "download_GBps": round(dn_bytes / last["download_ms"] / 1e6, 2)}))


if __name__ == "__main__":
    main()
