export PIRRT_WATCHDOG_MS=20000
timeout 120 python tools/debug_parity.py 2 6000 30 1 cfg2 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -5
PIRRT_BENCH_VERBOSE=1 python bench.py --graph-cache /tmp/g1m.npz --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r1c.json 2> gpurun_out/bench_r1c.err; cat gpurun_out/bench_r1c.json; grep -c step gpurun_out/bench_r1c.err
