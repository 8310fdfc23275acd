for dbg in 0 1 4 8 16 5 13; do
  SPD_DBG=$dbg SPD_LIB=tools/libspider_devel.so timeout 300 python tools/time_cfg.py B9 B27 B49 2>&1 | sed "s/^/dbg=$dbg /" | cut -c1-60
done
