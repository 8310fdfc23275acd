#!/bin/bash
# One-box A/B of three library builds (profiles/r02_m64_ct.txt):
#   tools/libspider_old.so   : the sources of commit 4694419 (before the M = 64 MMAs), built with the nvcc
#                              lines of tools/build_variant.sh from a `git archive 4694419` checkout
#   tools/libspider_nom64.so : tools/build_variant.sh nom64 -DSPD_NO_M64
#   the in-tree library
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for rep in 1 2; do
for lib in tools/libspider_old.so tools/libspider_nom64.so paper_2506_22035_b200/libspider.so; do
  SPD_LIB=$PWD/$lib timeout 200 python tools/m64_ab.py 3 B27 B9 2>&1 | grep -E "short|Error|error" | cut -c1-220
done; done
for lib in tools/libspider_old.so paper_2506_22035_b200/libspider.so; do
  SPD_LIB=$PWD/$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab_launch_$(basename $lib .so).csv python tools/prof_step.py B27 6 > /dev/null 2>&1
  grep spider_step gpurun_out/ab_launch_$(basename $lib .so).csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' '; echo " <- $lib"
done
