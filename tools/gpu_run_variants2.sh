test -f /tmp/g1m.npz || python bench.py --graph-cache /tmp/g1m.npz --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
for lib in "" paper_2003_04920_b200/lib/libpirrt_t512_b3.so paper_2003_04920_b200/lib/libpirrt_t256_b6.so paper_2003_04920_b200/lib/libpirrt_t256_b8.so; do
  PIRRT_LIB=$lib timeout 300 python tools/variant_probe.py 2>&1 | tail -1
done
