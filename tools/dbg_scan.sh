#!/bin/bash
# role-elimination scan (dev aid): which role limits the step time
for v in 0 1 2 4 8 6 14; do echo "== SPD_DBG=$v"; SPD_DBG=$v timeout 300 python tools/quick_time.py 2>&1 | sed -n '1p;3p'; done
