for i in 1 2; do
for lib in paper_2506_22035_b200/libspider.so tools/libspider_prevk.so; do
for c in B9 B27; do
SPD_LIB=$lib timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib $c', d['value'], d['clocks']['sm_mhz'])"
done; done; done
