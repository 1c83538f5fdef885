"""Generate the golden fixtures in tests/golden/ by running the UNMODIFIED
reference library (oracle/_ref/libthiim_ref.so, compiled from
/root/reference/proj/src by oracle/Makefile).  Run in the dev container:

    python tests/golden/make_golden.py

Each fixture stores the case definition, SHA-256 digests of the 40 input
arrays (so a test can confirm it rebuilt the same inputs), and the 12 output
field arrays after `steps` calls of the reference's run_naive.  Inputs are
rebuilt by the tests (generator / build_benchmark_problem restatement), so
only outputs are stored.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

CASES = [
    # name, dims, kind, seed, steps
    ("random_8x6x5_s3", (8, 6, 5), "random", 3, 3),
    ("random_13x4x9_s7", (13, 4, 9), "random", 7, 2),
    ("benchmark_8x8x8", (8, 8, 8), "benchmark", 0, 4),
    ("layered_6x6x12_s5", (6, 6, 12), "layered", 5, 2),
]


def build_inputs(dims, kind, seed):
    if kind == "random":
        return O.c_generate(dims, seed)
    if kind == "layered":
        return O.c_generate(dims, seed, layered=True)
    if kind == "benchmark":
        return O.ref_benchmark_problem(dims)
    raise ValueError(kind)


def digest(arrays):
    return [hashlib.sha256(a.tobytes()).hexdigest() for a in arrays]


def main():
    O.build()
    if not O.ref_available():
        raise SystemExit("oracle/_ref not built: needs /root/reference")
    index = []
    for name, dims, kind, seed, steps in CASES:
        arrays = build_inputs(dims, kind, seed)
        meta = {"name": name, "dims": dims, "kind": kind, "seed": seed, "steps": steps,
                "input_sha256": digest(arrays), "generator": "reference run_naive (oracle/_ref)"}
        O.ref_run_naive(dims, arrays, steps, 1)
        np.savez_compressed(os.path.join(HERE, name + ".npz"),
                            fields=np.stack(arrays[:12]), meta=json.dumps(meta))
        index.append(meta)
        print("wrote", name)
    with open(os.path.join(HERE, "index.json"), "w") as f:
        json.dump(index, f, indent=1)


if __name__ == "__main__":
    main()
