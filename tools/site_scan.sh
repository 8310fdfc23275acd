# which DEVEL-only runtime check changes B9's step time (isolating variants)
for i in 1 2; do
for v in prod devel m0 m1 m4 m8 tr; do
  lib=paper_2506_22035_b200/libspider.so; [ $v != prod ] && lib=tools/libspider_$v.so
  SPD_LIB=$lib timeout 300 python tools/time_cfg.py B9 W 2>&1 | sed "s/^/$v /" | cut -c1-60
done; done
