export GRAPH_CACHE=/tmp/g1m.npz
PIRRT_LIB=paper_2003_04920_b200/lib/libpirrt_trace.so timeout 600 python tools/cold_trace.py > gpurun_out/s2f_cold.log 2>&1
sed -n '/== rep 0/,$p' gpurun_out/s2f_cold.log | grep -v "^improve" | head -150
