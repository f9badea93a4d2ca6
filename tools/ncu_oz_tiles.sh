# DRAM bytes / duration / clock of the fp64 Ozaki environment GEMM under tiling / order variants
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second,lts__t_bytes.sum
for v in "bal:" "norot:TRALS_OZ_NOROT=1" "fix:TRALS_OZ_FIXED_TILES=1" "fixnorot:TRALS_OZ_FIXED_TILES=1 TRALS_OZ_NOROT=1"; do
  n=${v%%:*}; e=${v#*:}
  env $e ncu --metrics $M --clock-control none -k regex:oz8_kernel -c 1 --csv python tools/oz_probe64.py 25600 25600 20 1 > gpurun_out/ncu_$n.csv 2>&1
  echo "$n $(grep oz8 gpurun_out/ncu_$n.csv | awk -F'","' '{printf "%s=%s ", $(NF-2), $NF}')"
done
