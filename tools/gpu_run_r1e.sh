export PIRRT_WATCHDOG_MS=20000
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 20 python tools/debug_parity.py 2 6000 30 1 cfg2 2>&1 | tail -60
