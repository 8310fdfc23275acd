# producer scheduling variants (SPD_PROD_GUARD) against production
for i in 1 2; do
for v in prod es1 es2 eo; do
  lib=paper_2506_22035_b200/libspider.so; [ $v != prod ] && lib=tools/libspider_$v.so
  SPD_LIB=$lib timeout 300 python tools/time_cfg.py B9 W B27 B49 2>&1 | sed "s/^/$v /" | cut -c1-60
done; done
