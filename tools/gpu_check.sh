set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv | tail -1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_s2.log 2>&1; tail -3 gpurun_out/pytest_gpu_s2.log
timeout 600 python tools/quick_time.py persistent generic 2>&1 | tail -20
timeout 900 python bench.py > gpurun_out/bench_B9_s2.json 2> gpurun_out/bench_B9_s2.err; tail -1 gpurun_out/bench_B9_s2.json
