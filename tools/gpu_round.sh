#!/bin/bash
# One measurement session: smoke, gpu tests, bench lines (+reference arm),
# ncu launch lists + one full capture per config.
# usage: tools/gpu_round.sh <tag> [configs...]
set -u
TAG=${1:-r01}; shift || true
CONFIGS=${@:-B9 B49 B27 W}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $OUT/nvsmi_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; tail -1 $OUT/smoke_$TAG.log
timeout 900 python -m pytest tests -q -m gpu > $OUT/pytest_gpu_$TAG.log 2>&1; tail -1 $OUT/pytest_gpu_$TAG.log
timeout 600 python bench.py --impl reference > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err; tail -1 $OUT/bench_ref_$TAG.json | cut -c1-200
for c in $CONFIGS; do
  extra="--no-cpu-baseline --no-e2e"; [ "$c" = "B9" ] && extra=""
  timeout 900 python bench.py --config $c $extra > $OUT/bench_${c}_$TAG.json 2> $OUT/bench_${c}_$TAG.err; tail -1 $OUT/bench_${c}_$TAG.json | cut -c1-300
done
for c in $CONFIGS; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_${c}_$TAG.csv python tools/prof_step.py $c 6 > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:spider_step -s 3 -c 1 -o $OUT/prof_${c}_$TAG -f python tools/prof_step.py $c 5 > $OUT/ncu_${c}_$TAG.log 2>&1; tail -1 $OUT/ncu_${c}_$TAG.log
  python tools/ncu_summary.py $OUT/prof_${c}_$TAG.ncu-rep > $OUT/ncusum_${c}_$TAG.txt 2>&1
  # gpurun brings back <= 64 MiB: keep the full report of the first config only
  [ "$c" = "B9" ] || rm -f $OUT/prof_${c}_$TAG.ncu-rep
done
ls -la $OUT | tail -30
