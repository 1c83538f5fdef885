# A/B of the TBLOCK kernel across worktrees (one box): DRAM bytes + duration
# of one-wave exact-tile passes, and short-run MLUP/s
for i in 1 2; do
 for wt in build/wt_8c88876 .; do
  tag=$(basename $wt)
  opt="252x176x512:z_chunk=512"; [ "$wt" = . ] && opt="252x176x512:z_chunk=512,schedule=1"
  (cd $wt && ncu --kernel-name regex:k_tblock --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none --csv --log-file $OLDPWD/gpurun_out/r02n_${tag}_$i.csv python tools/traffic_probe.py $opt > /dev/null 2>&1)
 done
done
for wt in build/wt_8c88876 .; do
  opt="252x176x512:z_chunk=512"; [ "$wt" = . ] && opt="252x176x512:z_chunk=512,schedule=1"
  (cd $wt && python tools/traffic_probe.py $opt $opt 512x512x512 512x512x512 2>&1 | grep mlups | sed "s|^|$wt |")
done
