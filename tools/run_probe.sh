#!/bin/bash
# Runs every probe variant in its own process (a bad layout may trap the context).
cd "$(dirname "$0")"
mkdir -p ../gpurun_out
for v in 0 1 2 3 4; do timeout 60 ./umma_sp_probe $v; echo "exit=$?"; done 2>&1 | tee ../gpurun_out/probe.log
