#!/bin/bash
for v in 0 1 2 3 4 6; do echo "== SPD_PREFETCH=$v"; SPD_PREFETCH=$v timeout 300 python tools/quick_time.py 2>&1 | tail -4; done
