#!/bin/bash
# B27 re-tune after the M = 64 change: tools/time_cfg.py per build variant (tools/build_variant.sh), two rounds.
for rep in 1 2; do
for lib in paper_2506_22035_b200/libspider.so tools/libspider_pw5.so tools/libspider_ig5.so tools/libspider_ig10.so tools/libspider_nacc3.so; do
  echo -n "$(basename $lib) "; SPD_LIB=$PWD/$lib timeout 200 python tools/time_cfg.py B27 2>&1 | tail -1
done; done
