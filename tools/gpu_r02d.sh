# full GPU tests on the new defaults, default bench line, generic-path PW scan
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_r02d.log 2>&1; tail -3 gpurun_out/pytest_gpu_r02d.log
timeout 900 python bench.py > gpurun_out/bench_r02d.json 2> gpurun_out/bench_r02d.err; tail -1 gpurun_out/bench_r02d.json | cut -c1-300
for v in base gen4 gen6; do
  lib=paper_2506_22035_b200/libspider.so; [ $v != base ] && lib=tools/libspider_$v.so
  SPD_LIB=$lib timeout 300 python tools/time_cfg.py B25 2>&1 | sed "s/^/$v /"
done > gpurun_out/gen_pw_r02d.txt 2>&1; cat gpurun_out/gen_pw_r02d.txt
