# A/B: epilogue pairs (in-tree build) vs previous build (tools/libspider_prev.so); bench sampler / graph effects
timeout 300 python -m pytest tests -q -m gpu -x 2>&1 | tail -1
timeout 300 python tools/quick_time.py 2>&1 | tail -4
SPD_LIB=tools/libspider_prev.so timeout 300 python tools/quick_time.py 2>&1 | tail -4
for c in B9 B27; do
timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c stream', d['value'], d['clocks'])"
timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --graph 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c graph', d['value'])"
done
timeout 600 python bench.py --impl reference 2>/dev/null | tail -1 | cut -c1-300
