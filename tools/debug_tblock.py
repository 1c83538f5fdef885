import sys, numpy as np
sys.path.insert(0, '.')
import paper_1510_05218_b200 as P
from oracle import oracle as O
shape=(64,64,64)
d = P.GridDims(*shape)
s = P.generate_problem(d, P.GEN_RANDOM, 11)
w2 = P.clone_state(s); O.c_step(shape, w2.arrays, 2, threads=8)
for name, opts in [("fused BY16 ring6", dict(engine=P.ENGINE_FUSED, tile_y=116, z_chunk=8)),
                   ("tblock ring8", dict(engine=P.ENGINE_TBLOCK, z_chunk=8, debug=16)),
                   ("tblock", dict(engine=P.ENGINE_TBLOCK, z_chunk=8)),
                   ("tblock default", dict(engine=P.ENGINE_TBLOCK))]:
    tot = 0
    for rep in range(6):
        g = P.clone_state(s); P.run_gpu(g, 2, P.GpuOptions(**opts))
        tot += P.compare_states(g, w2).differing_values
    print(name, "mismatches over 6 runs:", tot, flush=True)
