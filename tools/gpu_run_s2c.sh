# cold-solve Improve timeline (trace build) + microbench reference
GRAPH_CACHE=/tmp/g1m.npz PIRRT_LIB=paper_2003_04920_b200/lib/libpirrt_trace.so timeout 900 python tools/cold_trace.py > gpurun_out/s2c_cold.log 2>&1; grep -E "^improve|^==" gpurun_out/s2c_cold.log | tail -24
