#!/bin/bash
# knob sweep of the product under the sustained (power-capped) bench
for rep in 1 2; do
for a in "" "--pol-mode 1" "--pol-mode 3" "--pol-mode 4" "--z-chunk 64" "--z-chunk 86" "--z-chunk 256" "--tile-y 14" "--min-blocks 1"; do
  timeout 300 python bench.py $a --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(repr('$a'),d['value'],d['roofline']['frac'],d['clocks']['sm_mhz'],d['clocks'].get('power_w'))"
done; done
