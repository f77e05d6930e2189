export PIRRT_WATCHDOG_MS=20000
timeout 200 python tools/debug_parity.py 2 6000 30 1 cfg2 2>&1 | tail -6
timeout 200 python tools/debug_parity.py 2 6000 30 1 cfg2 2>&1 | tail -3
