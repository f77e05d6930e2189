# section 8(d) suite at the current code + host facts
free -g | head -2; nproc; df -h /tmp | tail -1
timeout 2400 python tools/suite.py --out gpurun_out/suite_s2.json > gpurun_out/s2k_suite.log 2>&1; tail -5 gpurun_out/s2k_suite.log
PIRRT_BENCH_VERBOSE=1 python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench.npz > gpurun_out/s2k_bench.json 2> gpurun_out/s2k_bench.err; grep -E "step" gpurun_out/s2k_bench.err | head -30
