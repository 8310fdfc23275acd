timeout 600 python -m pytest -q -x tests/test_gpu_multidevice.py > gpurun_out/t_r02b.log 2>&1; tail -3 gpurun_out/t_r02b.log
timeout 300 python tools/e2e_scan.py B9 0 2 3 4 5 6 8 > gpurun_out/e2e_scan_B9.txt 2>&1; cat gpurun_out/e2e_scan_B9.txt
for v in base e2p4 e2p6 p6 p4; do
  lib=paper_2506_22035_b200/libspider.so; [ $v != base ] && lib=tools/libspider_$v.so
  SPD_LIB=$lib timeout 300 python tools/time_cfg.py B9 B27 B49 2>&1 | sed "s/^/$v /"
done > gpurun_out/variants_r02b.txt 2>&1; cat gpurun_out/variants_r02b.txt
