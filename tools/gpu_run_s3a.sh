export GRAPH_CACHE=/tmp/g1m.npz
for lib in libpirrt.so libpirrt_w8_8_4.so libpirrt_w8_4_5.so libpirrt_w32_2_4.so; do
  PIRRT_LIB=paper_2003_04920_b200/lib/$lib timeout 600 python tools/wide_probe.py 2>&1 | tail -1
done
