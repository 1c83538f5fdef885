#!/bin/bash
# ncu --set full of one TBLOCK round at configs[2]: an in-place view covering all
# of z (THIIM_INPLACE_TB=512, one sub-range) vs the whole-z ping-pong round
O=gpurun_out/vw; mkdir -p $O
THIIM_INPLACE_TB=512 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tblock_tm -s 20 -c 1 -o $O/view python bench.py --config c2 --engine tblock-inplace --no-e2e --no-cpu-baseline --steps 1 --warmup 0 --iters 8 > $O/v.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tblock_tm -s 20 -c 1 -o $O/whole python bench.py --config c2 --no-e2e --no-cpu-baseline --steps 1 --warmup 0 --iters 8 > $O/w.log 2>&1
