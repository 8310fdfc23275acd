for lib in paper_2506_22035_b200/libspider.so tools/libspider_n3.so tools/libspider_n2.so tools/libspider_a3.so tools/libspider_a2.so; do
echo "== $lib"; SPD_LIB=$lib timeout 300 python tools/quick_time.py 2>&1 | sed -n 3p
done
