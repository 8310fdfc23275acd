#!/bin/bash
# A/B of L2 cache-policy builds (tools/build_variant.sh l2h<v> -DSPD_L2_HINT=<v>) against the in-tree library.
for rep in 1 2; do
for lib in paper_2506_22035_b200/libspider.so tools/libspider_l2h1.so tools/libspider_l2h2.so tools/libspider_l2h3.so; do
  SPD_LIB=$PWD/$lib timeout 200 python tools/m64_ab.py 3 B9 B27 2>&1 | grep -E "short|Error|error" | cut -c1-60,84-240
done; done
for lib in paper_2506_22035_b200/libspider.so tools/libspider_l2h1.so tools/libspider_l2h2.so tools/libspider_l2h3.so; do
  for c in B9 B27; do
  SPD_LIB=$PWD/$lib timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/l2_$(basename $lib .so)_$c.csv python tools/prof_step.py $c 6 > /dev/null 2>&1
  echo "$c $lib"; grep spider_step gpurun_out/l2_$(basename $lib .so)_$c.csv | awk -F'","' '{print $(NF-2), $NF}' | tr -d '"' | tail -8 | tr '\n' ';'; echo
  done
done
