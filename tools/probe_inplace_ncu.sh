#!/bin/bash
# ncu launch list + one full capture of an in-place sub-range round at configs[2]
O=gpurun_out/ipn; mkdir -p $O
B="python bench.py --config c2 --engine tblock-inplace --no-e2e --no-cpu-baseline --steps 1 --warmup 3"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv $B > $O/l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tblock_tm -s 200 -c 1 -o $O/ip_round $B > $O/f.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tblock_tm -s 40 -c 1 -o $O/whole_round python bench.py --config c2 --no-e2e --no-cpu-baseline --steps 1 --warmup 3 > $O/f2.log 2>&1
