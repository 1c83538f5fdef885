o=gpurun_out/chunk
for zc in 0 256 128 64 0; do
  SWEEP_STEPS=40 timeout 300 python tools/grid_sweep.py 512x512x512:z_chunk=$zc >> ${o}_sweep.jsonl 2>>${o}.err
done
for zc in 0 256 128; do
  SWEEP_STEPS=2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none --csv --log-file ${o}_ncu_$zc.csv -k regex:k_tblock_tm python tools/grid_sweep.py 512x512x512:z_chunk=$zc > /dev/null 2>>${o}.err
done
echo done
