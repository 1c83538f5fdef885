# A/B of the array stride padding (THIIM_STRIDE_PAD elements) at configs[2]'s grid
o=gpurun_out/stride
for rep in 1 2; do
for pad in 0 16 64 256 1040 8208; do
  THIIM_STRIDE_PAD=$pad SWEEP_STEPS=100 timeout 300 python tools/grid_sweep.py 512x512x512 | sed "s/^/{\"pad\": $pad, \"rep\": $rep, \"r\": /; s/\$/}/" >> ${o}_sweep.jsonl 2>>${o}.err
done
done
echo done
