# energy per step (sustained, power-capped) and short-run time per library variant: bash tools/energy_scan.sh v1 v2 ...
for v in "$@"; do
  lib=paper_2506_22035_b200/libspider.so; [ $v != prod ] && lib=tools/libspider_$v.so
  for c in B9 B27; do
    echo "$v $c $(SPD_LIB=$lib python tools/power_probe.py $c 3 | grep energy)"
    sleep 4
  done
  SPD_LIB=$lib timeout 300 python tools/time_cfg.py B9 B27 2>&1 | sed "s/^/$v short /" | cut -c1-70
done
