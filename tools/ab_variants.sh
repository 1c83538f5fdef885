#!/bin/bash
# Interleaved A/B of library builds on one box:
#   tools/ab_variants.sh "<bench args>" REPS name=path.so [name=path.so ...]
# "product" = paper_1510_05218_b200/libthiim_gpu.so.  Prints name, MLUP/s, SM clock.
args=$1; reps=$2; shift 2
for i in $(seq "$reps"); do
  for v in "$@"; do
    name=${v%%=*}; lib=${v#*=}
    [ "$lib" = product ] && lib=paper_1510_05218_b200/libthiim_gpu.so
    timeout 600 env THIIM_LIB=$lib python bench.py $args --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 |
      python -c "import json,sys;d=json.loads(sys.stdin.read());print('$name',d['value'],d['roofline']['frac'],d['clocks']['sm_mhz'],d['clocks'].get('power_w'))"
  done
done
