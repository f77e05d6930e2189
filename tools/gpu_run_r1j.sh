export PIRRT_WATCHDOG_MS=20000
timeout 120 python tools/debug_parity.py 2 6000 30 1 cfg2 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q -p pytest_timeout --timeout 300 2>&1 | tail -8
python bench.py --graph-cache /tmp/g1m.npz --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r1b.json 2> gpurun_out/bench_r1b.err; cat gpurun_out/bench_r1b.json; tail -3 gpurun_out/bench_r1b.err
