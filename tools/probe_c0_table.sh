#!/bin/bash
# c0 (64^3 x 50) geometry sweep + ncu of one k_tblock_tm launch at c0, and an
# ncu capture of the table kernel at c3 (gpurun probe; outputs in gpurun_out/)
set -u
O=gpurun_out/c0
mkdir -p $O
B="python bench.py --config c0 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e"
for a in "" "--tile-y 12" "--tile-y 14" "--z-chunk 4" "--z-chunk 6" "--z-chunk 11" "--z-chunk 16" "--z-chunk 22" "--time-block 3" "--schedule 1"; do
  echo "== $a" >> $O/sweep.txt
  timeout 300 $B $a 2>>$O/sweep.err | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(j['value'], j['roofline']['frac'], j['clocks']['sm_mhz'], j['config'].get('engine'))" >> $O/sweep.txt
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --config c0 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_l.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tblock_tm -s 30 -c 1 -o $O/c0_tblock python bench.py --config c0 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1
echo done >> $O/sweep.txt
