#!/bin/bash
# Round-2 measurement session: smoke, gpu tests, default bench line (+ side
# configs, e2e, cpu baseline), reference arm, ncu launch lists + full captures.
# usage: tools/gpu_r2.sh <tag> [tests:0|1] [configs to profile...]
set -u
TAG=${1:-r02a}; shift || true
TESTS=${1:-1}; shift || true
CONFIGS=${@:-B9 B27}
FIRST=${CONFIGS%% *}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $OUT/nvsmi_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; tail -1 $OUT/smoke_$TAG.log
if [ "$TESTS" = "1" ]; then
  timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu_$TAG.log 2>&1; tail -3 $OUT/pytest_gpu_$TAG.log
fi
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; tail -1 $OUT/bench_$TAG.json | cut -c1-400
for c in $CONFIGS; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_${c}_$TAG.csv python tools/prof_step.py $c 6 > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:spider_step -s 3 -c 1 -o $OUT/prof_${c}_$TAG -f python tools/prof_step.py $c 5 > $OUT/ncu_${c}_$TAG.log 2>&1; tail -1 $OUT/ncu_${c}_$TAG.log
  python tools/ncu_summary.py $OUT/prof_${c}_$TAG.ncu-rep > $OUT/ncusum_${c}_$TAG.txt 2>&1
  # gpurun brings back <= 64 MiB: keep the full report of the first config only
  [ "$c" = "$FIRST" ] || rm -f $OUT/prof_${c}_$TAG.ncu-rep
done
ls -la $OUT | tail -30
