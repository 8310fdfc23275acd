#!/bin/bash
# variant scan (dev aid): SPD_TUNE selects stage configs, SPD_NTILE64 the 2D tile width
for v in 0 1; do echo "== SPD_TUNE=$v"; SPD_TUNE=$v timeout 300 python tools/quick_time.py 2>&1 | tail -4; done
for v in 0 1 2; do echo "== SPD_NTILE64 SPD_TUNE=$v"; SPD_NTILE64=1 SPD_TUNE=$v timeout 300 python tools/quick_time.py 2>&1 | head -1; done
echo "== 3D tune 2"; SPD_TUNE=2 timeout 300 python tools/quick_time.py 2>&1 | sed -n 3p
