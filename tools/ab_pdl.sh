#!/bin/bash
# A/B: TBLOCK rounds as programmatic dependent launches vs ordinary launches
O=gpurun_out/pdl; mkdir -p $O
run() {  # label env... -- bench args
  local label=$1; shift
  echo -n "$label " >> $O/ab.txt
  env "$@" python bench.py --no-e2e --no-cpu-baseline --steps 3 --warmup 3 $BARGS 2>>$O/err.txt | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(j['value'], j['roofline']['frac'], j['clocks']['sm_mhz'], j['clocks'].get('power_w'))" >> $O/ab.txt
}
for rep in 1 2; do
  BARGS="--config c2" run c2_pdl X=1
  BARGS="--config c2" run c2_nopdl THIIM_NO_PDL=1
  BARGS="--config c2 --engine tblock-inplace" run c2ip_pdl X=1
  BARGS="--config c2 --engine tblock-inplace" run c2ip_nopdl THIIM_NO_PDL=1
  BARGS="--config c1" run c1_pdl X=1
  BARGS="--config c1" run c1_nopdl THIIM_NO_PDL=1
  BARGS="--config c0" run c0_pdl X=1
  BARGS="--config c0" run c0_nopdl THIIM_NO_PDL=1
done
