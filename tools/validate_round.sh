set -x
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/f_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/f_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/f_smoke.log
timeout 400 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/f_reference_arm.json 2> gpurun_out/f_ref.err
: > gpurun_out/f_configs.jsonl
for a in "--config c0" "--config c2" "--config c3" "--config c3 --coeff table" "--config c4"; do
  timeout 900 python bench.py $a 2>>gpurun_out/f_configs.err | tail -1 >> gpurun_out/f_configs.jsonl
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tblock_table -c 1 -o gpurun_out/f_table python bench.py --config c3 --coeff table --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/f_ncu_table.log 2>&1
echo done
