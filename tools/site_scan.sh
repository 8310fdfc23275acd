# library variants against production (interleaved rounds; time_cfg cools down before each config)
# usage: bash tools/site_scan.sh "CONFIGS" variant...
CFGS=$1; shift
for i in 1 2; do
for v in prod "$@"; do
  lib=paper_2506_22035_b200/libspider.so; [ $v != prod ] && lib=tools/libspider_$v.so
  SPD_LIB=$lib timeout 300 python tools/time_cfg.py $CFGS 2>&1 | sed "s/^/$v /" | cut -c1-60
done; done
