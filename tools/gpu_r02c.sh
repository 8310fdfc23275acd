# producer-warp scan per geometry + streamed e2e with 1/2 compute streams
for v in base pw2 pw3 pw5; do
  lib=paper_2506_22035_b200/libspider.so; [ $v != base ] && lib=tools/libspider_$v.so
  SPD_LIB=$lib timeout 300 python tools/time_cfg.py B27 B49 B9 2>&1 | sed "s/^/$v /"
done > gpurun_out/pw_r02c.txt 2>&1; cat gpurun_out/pw_r02c.txt
SPD_PROD_WARPS_NOTE=generic timeout 300 python tools/time_cfg.py B25 | sed "s/^/base /" >> gpurun_out/pw_r02c.txt
for c in 1 2; do SPD_STREAM_COMPUTE=$c timeout 300 python tools/e2e_scan.py B9 3 4 6 8 | sed "s/^/compute=$c /"; done > gpurun_out/e2e_scan2.txt 2>&1; cat gpurun_out/e2e_scan2.txt
timeout 300 python tools/e2e_scan.py W 0 4 6 8 >> gpurun_out/e2e_scan2.txt 2>&1; tail -4 gpurun_out/e2e_scan2.txt
