export PIRRT_WATCHDOG_MS=20000
DBG_GRID=1 timeout 200 python tools/debug_parity.py 2 6000 30 1 cfg2 2>&1 | tail -6
DBG_GRID=2 timeout 200 python tools/debug_parity.py 2 6000 30 1 cfg2 2>&1 | tail -6
