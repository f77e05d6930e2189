# wide Improve: parity + cold-solve variants
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s2d_tests.log 2>&1; tail -4 gpurun_out/s2d_tests.log
export GRAPH_CACHE=/tmp/g1m.npz
PIRRT_WIDE_TASKS=0 timeout 600 python tools/wide_probe.py 2>&1 | tail -1
for v in 16_2_6 32_2_6 16_4_4 32_1_8 8_2_6 16_2_5; do
  PIRRT_LIB=paper_2003_04920_b200/lib/libpirrt_w$v.so timeout 600 python tools/wide_probe.py 2>&1 | tail -1
done
