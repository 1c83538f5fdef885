# End-of-session validation on one B200 (gpurun): GPU tests, smoke, the default
# bench line (configs[2]) and the reference arm, the other configs, the launch
# list of the bench command with DRAM bytes (per-pass traffic), and one
# `ncu --set full` capture of a k_tblock_tm round at configs[2].
# usage: bash tools/validate_round.sh TAG
tag=${1:-f}
o=gpurun_out/$tag
timeout 1500 python -m pytest tests -q -m gpu > ${o}_tests.log 2>&1; echo tests_rc=$? >> ${o}_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > ${o}_smoke.log 2>&1; echo smoke_rc=$? >> ${o}_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > ${o}_bench.json 2> ${o}_bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > ${o}_reference_arm.json 2> ${o}_ref.err
: > ${o}_configs.jsonl
for a in "--config c0" "--config c1" "--config c3 --no-e2e" "--config c3 --coeff table" "--config c4 --no-e2e"; do
  timeout 900 python bench.py $a --no-cpu-baseline 2>>${o}_configs.err | tail -1 >> ${o}_configs.jsonl
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none --csv --log-file ${o}_launches.csv python bench.py --steps 1 --warmup 0 --iters 20 --no-e2e --no-cpu-baseline > ${o}_ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tblock_tm -s 6 -c 1 -o ${o}_tblock_c2 python bench.py --steps 1 --warmup 0 --iters 4 --no-e2e --no-cpu-baseline > ${o}_ncu_full.log 2>&1
echo done
