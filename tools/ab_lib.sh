#!/bin/bash
# A/B of two builds of libthiim_gpu.so on one box (THIIM_LIB selects the
# library): bash tools/ab_lib.sh OLD.so OUTDIR "bench args 1" "bench args 2" ...
old=$1; out=$2; shift 2
mkdir -p $out
for rep in 1 2; do
  for args in "$@"; do
    for lib in $old paper_1510_05218_b200/libthiim_gpu.so; do
      echo -n "$(basename $lib) | $args | " >> $out/ab.txt
      THIIM_LIB=$lib python bench.py $args --no-cpu-baseline --no-e2e 2>>$out/err.txt | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(j['value'], j['roofline']['frac'], j['clocks']['sm_mhz'], j['clocks'].get('power_w'))" >> $out/ab.txt
    done
  done
done
